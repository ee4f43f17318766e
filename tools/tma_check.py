import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2512_12151_b200 import scenes
from paper_2512_12151_b200.device import to_dev, empty, to_host
system, state, params = scenes.c4_scene(n=20)
dev = system.device
x = to_dev(state.x); xt = to_dev(state.x + 1e-4)
g = empty((system.n_vertices, 3))
dev.assemble(None, x, xt, 1.0, 1e-3, 0.01, True, g)
p = torch.from_numpy(np.random.default_rng(0).standard_normal((system.n_vertices, 3))).cuda()
y = empty((system.n_vertices, 3)); dev.matvec(p, y)
np.save(sys.argv[1], to_host(y))
