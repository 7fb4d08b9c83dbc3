"""Parity helpers shared by the GPU tests (tolerances of BASELINE.json north_star, readings Q22/Q23)."""
import numpy as np

TOL = 1e-10      # mu, Sigma relative error (north_star)
BAND = 1e-9      # tie band for subsets / flags (north_star)


def rel_sigma(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def rel_mu(a, b, Sigma):
    """||a - b|| / max(||b||, sqrt(tr Sigma / p)) (reading Q22)."""
    b = np.asarray(b)
    den = max(np.linalg.norm(b), np.sqrt(np.trace(Sigma) / len(b)))
    return float(np.linalg.norm(np.asarray(a) - b) / den)


def assert_flags_equal(gpu_flags, oracle_flags, oracle_rd2, cutoff2, band=BAND):
    """Identical except rows whose RD lies within band (relative) of the cut-off c_p."""
    g = np.asarray(gpu_flags).astype(bool)
    o = np.asarray(oracle_flags).astype(bool)
    d = np.sqrt(np.maximum(oracle_rd2, 0))
    cp = np.sqrt(cutoff2)
    exempt = np.abs(d - cp) <= band * cp
    bad = (g != o) & ~exempt
    assert not bad.any(), f"{bad.sum()} flag mismatches outside the tie band (first {np.nonzero(bad)[0][:5]})"
    return int(exempt.sum())


def assert_subset_equal(gpu_mask, oracle_H, d2_oracle, h, band=BAND):
    """h-subset identical except rows whose distance is within band of the h-th distance."""
    g = np.asarray(gpu_mask).astype(bool)
    o = np.zeros_like(g)
    o[np.asarray(oracle_H)] = True
    d = np.sqrt(np.maximum(d2_oracle, 0))
    dh = np.sort(d)[h - 1]
    exempt = np.abs(d - dh) <= band * dh
    bad = (g != o) & ~exempt
    assert not bad.any(), f"{bad.sum()} subset mismatches outside the tie band"
    assert g.sum() == h
