#!/bin/bash
# launch times of the select kernels (config 4) under RTD_SEL_CTAS_PER_SM = 1 2 4 8
for c in 1 2 4 8; do
  RTD_SEL_CTAS_PER_SM=$c ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sel" --csv \
    --log-file gpurun_out/sel_$c.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
done
