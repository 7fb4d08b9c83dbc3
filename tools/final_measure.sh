#!/bin/bash
# Round-end measurement set (one gpurun call): GPU tests, smoke, the default bench line, the reference arm,
# launch lists of config 4 and config 5.  Outputs under gpurun_out/final/.
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_reference.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launch4.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launch5.csv \
  python bench.py --config 5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
