"""Run tools/fp64_peak on the GPU box and write profiles/fp64_peak.json (best DMMA / DFMA of the reps)."""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = subprocess.run([os.path.join(ROOT, "tools", "fp64_peak")], capture_output=True, text=True, check=True).stdout
dmma = max(float(x) for x in re.findall(r"DMMA m8n8k4: ([0-9.]+) TFLOP/s", out))
dfma = max(float(x) for x in re.findall(r"DFMA: ([0-9.]+) TFLOP/s", out))
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,name", "--format=csv,noheader"],
                     capture_output=True, text=True).stdout.strip()
res = {"dmma_tflops": dmma, "dfma_tflops": dfma, "clocks_after": clk, "raw": out.strip().splitlines(),
       "how": "tools/fp64_peak.cu: 148*8 CTAs x 256 threads, 20000 iterations of 8 independent DMMA m8n8k4 "
              "(16 DFMA) chains per warp (thread), best of 3 CUDA-event-timed launches"}
json.dump(res, open(os.path.join(ROOT, sys.argv[1] if len(sys.argv) > 1 else "profiles/fp64_peak.json"), "w"), indent=1)
print(json.dumps(res))
