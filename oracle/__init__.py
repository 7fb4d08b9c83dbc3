"""CPU oracle for RT-DetMCD (arXiv 1910.05615) — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 implementation of what the paper
defines, written from /root/reference/PAPER.md (cited as PAPER.md:<line>,
section / equation).  It shares no code with the CUDA path and never imports
it.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline`
leg (and `bench.py --impl reference`) may import or call anything in here;
the product package `paper_1910_05615_b200` must never route through it.

Modules
  chi2       chi-square CDF / quantile, consistency factor c(alpha, p)
  numerics   small dense linear algebra (p <= 40)
  unimcd     univariate raw / reweighted MCD (exact window argmin)
  initial    wrapping S~1 and LR-GSSCM S~2
  refine     refinement of the initial estimates
  cstep      concentration steps
  parallel   partition, aggregation (median, KL, pooling)
  fit        the whole RT-DetMCD fit (serial IDC and blocked IDCP_q) + flag

Every function is pinned by `tests/test_oracle_*.py` (-m "not gpu") against
closed forms, paper-printed values, brute force or invariants.  Functions
without such a pin say "parity unpinned" in their docstring (none at present).
"""
