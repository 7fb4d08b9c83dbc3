"""Host-side launch trace of config-5 cold fits (RTD_TRACE_HOST=1 prints the deltas at exit)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1910_05615_b200 import api, datagen  # noqa: E402

bs = [datagen.make_config(5, batch=b) for b in range(8)]
Xs = [torch.from_numpy(b.X).cuda() for b in bs]
for X, b in zip(Xs, bs):
    api.fit(X, h=b.h, log_transform=b.log_transform, outputs=("flags",))
torch.cuda.synchronize()
print("done")
