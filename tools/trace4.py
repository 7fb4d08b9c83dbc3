"""Host-side launch trace of one config-4 fit after a warm-up (RTD_TRACE_HOST=1 prints the deltas at exit)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1910_05615_b200 import api, datagen  # noqa: E402

d = datagen.make_config(4)
X = torch.from_numpy(d.X).cuda()
for _ in range(2):
    api.fit(X, h=int(0.75 * X.shape[0]), q=8, partition=1, outputs=("flags",))
torch.cuda.synchronize()
print("done")
