"""One FSEP layer step at BASELINE configs[0] shape (8 virtual ranks) for compute-sanitizer.

Usage: python tools/sanitize_step.py [ce]   ("ce": virtual copy-engine mode)"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
if len(sys.argv) > 1 and sys.argv[1] == "ce":
    os.environ["FSEP_COMM"] = "ce"

import numpy as np
import torch

from oracle import layer_oracle as LO
from paper_2602_11686_b200 import planner as PL
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec

N, E, K, H, F, T, C = 8, 8, 2, 256, 512, 512, 2
g = torch.Generator().manual_seed(42)
layer = FsepLayer(LayerSpec(E, K, H, F, T, C, world=N, virtual=True))
for e in range(E):
    layer.load_expert(e, (torch.randn(F, H, generator=g) / 16).bfloat16().cuda(),
                      (torch.randn(F, H, generator=g) / 16).bfloat16().cuda(),
                      (torch.randn(H, F, generator=g) / 22).bfloat16().cuda())
layer.load_router((torch.randn(E, H, generator=g) * 0.02).bfloat16().cuda())
rng = np.random.default_rng(1)
bias = torch.from_numpy(np.concatenate([LO.make_bias(rng, T, E, 1.2) for _ in range(N)])).cuda()
x = torch.randn(N * T, H, generator=g).bfloat16().cuda()
dy = (torch.randn(N * T, H, generator=g) * 0.1).bfloat16().cuda()
y, dx = torch.empty_like(x), torch.empty_like(x)
for A in (PL.even_replication_layout(N, E, C), PL.static_ep_layout(N, E, C)):
    layer.set_layout(A)
    layer.forward(x, bias, T, y)
    layer.backward(dy, dx)
torch.cuda.synchronize()
layer.close()
print("sanitize step ok")
