"""The C-ABI library loads and exports every symbol include/rtdetmcd.h declares (CPU-only checks).

Host-side scalar numerics of the product library (chi2 quantile, c(alpha),
the q rule) are compared with the oracle here; no CUDA work is launched.
"""
import ctypes
import os
import re

import pytest

from oracle.chi2 import chi2_quantile as o_chi2, consistency_factor as o_cf
from oracle.parallel import choose_q as o_choose_q

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rtdetmcd.h")
LIB = os.path.join(ROOT, "paper_1910_05615_b200", "libpaper_1910_05615_b200.so")


def _declared():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rtdetmcd_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def so():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def test_header_declares_expected_entry_points():
    names = _declared()
    for must in ("rtdetmcd_create", "rtdetmcd_fit", "rtdetmcd_flag", "rtdetmcd_last_error", "rtdetmcd_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol(so):
    missing = [n for n in _declared() if not hasattr(so, n)]
    assert not missing, missing


def test_binding_covers_every_symbol():
    from paper_1910_05615_b200._lib import EXPORTS
    assert sorted(EXPORTS) == _declared()


def test_host_numerics_match_oracle(so):
    from paper_1910_05615_b200 import api
    for p in (1, 2, 5, 8, 10, 20, 40):
        for u in (0.5, 0.75, 0.975, 0.999):
            assert api.chi2_quantile(u, p) == pytest.approx(o_chi2(u, p), rel=1e-13)
        for a in (0.5, 0.500001, 0.6, 0.75, 0.975):
            assert api.consistency_factor(a, p) == pytest.approx(o_cf(a, p), rel=1e-12)
    for n, p, w in ((2 ** 16, 4, 4096), (2 ** 19, 8, 8192), (8_000_000, 40, 4096), (1000, 5, 4096)):
        assert api.choose_q(n, p, w) == o_choose_q(n, p, w)


def test_library_has_no_undefined_internal_symbols(so):
    """Every rtd:: symbol the library references is defined in it (a shared object links with
    undefined symbols and would only fail at load / first call)."""
    import shutil
    import subprocess
    if not shutil.which("nm"):
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-D", "--undefined-only", LIB], capture_output=True, text=True).stdout
    bad = [ln for ln in out.splitlines() if "rtd" in ln or "rtdetmcd" in ln]
    assert not bad, bad


def test_wrap_tanh_table_accuracy():
    """The device tanh table of the wrapping function's tanh branch (csrc/tanh_table.h, PAPER.md:478-486:
    argument q2 (c - |z|) in [0, 2.155]) evaluated as k_moments_tma evaluates it (interval rint(x / W),
    Estrin) is within 3 ulp of numpy's tanh on a dense grid and at the interval ends (reading R28)."""
    import numpy as np
    txt = open(os.path.join(ROOT, "paper_1910_05615_b200", "csrc", "tanh_table.h")).read()
    ni = int(re.search(r"#define RTD_TANH_NI (\d+)", txt).group(1))
    nc = int(re.search(r"#define RTD_TANH_NC (\d+)", txt).group(1))
    body = txt[txt.index("{") + 1:txt.index("};")]
    a = np.array([float.fromhex(t) for t in body.replace("\n", " ").split(",") if t.strip()]).reshape(ni, nc)
    w = 2.16 / 32
    x = np.concatenate([np.linspace(0.0, 0.862 * 2.5, 200_001), (np.arange(ni) + 0.5) * w])
    x = x[x <= 0.862 * 2.5]
    j = np.minimum(np.rint(x * (1.0 / w)).astype(np.int64), ni - 1)
    v = x - j * w
    c = a[j]
    v2 = v * v
    v4 = v2 * v2
    p = [c[:, k] + c[:, k + 1] * v for k in (0, 2, 4, 6, 8)]
    q0, q1, q2 = p[0] + p[1] * v2, p[2] + p[3] * v2, p[4] + c[:, 10] * v2
    y = (q0 + q1 * v4) + q2 * (v4 * v4)
    ref = np.tanh(x)
    ulp = np.spacing(np.maximum(np.abs(ref), np.finfo(float).tiny))
    assert y[0] == 0.0
    assert (np.abs(y - ref)[1:] / ulp[1:]).max() <= 3.0


def test_wrap_tanh_table_matches_its_generator():
    """csrc/tanh_table.h holds exactly the coefficients tools/gen_tanh_table.py derives (mpmath Taylor
    coefficients about c_j = j W rounded to fp64): the table is not hand-edited."""
    import importlib.util
    import numpy as np
    spec = importlib.util.spec_from_file_location("gen_tanh_table", os.path.join(ROOT, "tools", "gen_tanh_table.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    txt = open(os.path.join(ROOT, "paper_1910_05615_b200", "csrc", "tanh_table.h")).read()
    body = txt[txt.index("{") + 1:txt.index("};")]
    a = np.array([float.fromhex(t) for t in body.replace("\n", " ").split(",") if t.strip()])
    assert np.array_equal(a, gen.coeffs().ravel())
