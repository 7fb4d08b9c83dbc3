"""Debug helper: run one config-4 fit with RTD_DEBUG_PRUNED=1 and summarise the pruned-path statuses."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1910_05615_b200 import api, datagen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
d = datagen.make_config(cfg)
X = torch.from_numpy(d.X).cuda()
g = api.fit(X, h=d.h, q=d.q, seed=191005615, log_transform=d.log_transform, outputs=("flags",))
print("chosen", g.block_chosen, "steps", g.start_steps)
