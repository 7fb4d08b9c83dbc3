import sys, torch
from paper_1910_05615_b200 import api, datagen
d = datagen.make_config(int(sys.argv[1]))
X = torch.from_numpy(d.X).cuda()
g = api.fit(X, h=d.h, q=int(sys.argv[2]), seed=191005615, log_transform=d.log_transform, outputs=())
print(g.start_steps, g.block_chosen)
