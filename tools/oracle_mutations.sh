#!/usr/bin/env bash
# Mutation check of the oracle pins: each mutation below must make at least one
# -m "not gpu" oracle-pin test fail.  Run from the repo root: bash tools/oracle_mutations.sh
set -u
run() { # name file from to
  d=/tmp/mut_$1; rm -rf $d; mkdir -p $d
  cp -r oracle tests paper_1910_05615_b200 $d/ 2>/dev/null
  rm -f $d/paper_1910_05615_b200/*.so
  python - "$d/$2" "$3" "$4" <<'PY'
import sys; f,a,b=sys.argv[1:]; s=open(f).read(); assert a in s, (f,a); open(f,'w').write(s.replace(a,b,1))
PY
  (cd $d && timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_oracle_unimcd.py tests/test_oracle_initial.py tests/test_oracle_refine_cstep.py tests/test_oracle_parallel.py tests/test_oracle_fit.py -m "not gpu" 2>&1 | tail -2 | sed "s/^/$1: /")
}
run refine_half oracle/refine.py "mu = Sig_half @ mt" "mu = Sig_mhalf @ mt"
run refine_raw oracle/refine.py "unimcd_reweighted(T[:, j]).scale ** 2" "unimcd_raw(T[:, j], T.shape[0] // 2 + 1).var"
run refine_raw_loc oracle/refine.py "unimcd_reweighted(Zt[:, j]).loc" "unimcd_raw(Zt[:, j], Zt.shape[0] // 2 + 1).loc"
run rew_factor oracle/fit.py "Sigma_rew = consistency_factor(quantile, p) * (D.T @ D) / (k - 1)" "Sigma_rew = (D.T @ D) / (k - 1)"
run margin oracle/unimcd.py "err = 2.0 * err + 1e-300" "err = 0.0 * err"
