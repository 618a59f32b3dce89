import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import layer_oracle as LO
from paper_2602_11686_b200 import planner as PL
from paper_2602_11686_b200.layer import FsepLayer, LayerSpec
N, E, K, H, F, T, C = 8, 8, 2, int(os.environ.get("HH", 4096)), int(os.environ.get("FF", 14336)), 512, 2
layer = FsepLayer(LayerSpec(E, K, H, F, T, C, world=N, virtual=True, copy_engine=True))
g = torch.Generator(device="cuda").manual_seed(3)
for e in range(E):
    layer.load_expert(e, (torch.randn(F, H, device="cuda", generator=g) / 64).bfloat16(), (torch.randn(F, H, device="cuda", generator=g) / 64).bfloat16(), (torch.randn(H, F, device="cuda", generator=g) / 64).bfloat16())
layer.load_router((torch.randn(E, H, device="cuda", generator=g) * 0.02).bfloat16())
layer.set_layout(PL.even_replication_layout(N, E, C))
rng = np.random.default_rng(1)
bias = torch.from_numpy(np.concatenate([LO.make_bias(rng, T, E, 1.2) for _ in range(N)])).cuda()
x = torch.randn(N * T, H, device="cuda").bfloat16(); dy = torch.randn(N * T, H, device="cuda").bfloat16() * 0.1
y, dx = torch.empty_like(x), torch.empty_like(x)
for i in range(2):
    t0 = time.time()
    layer.forward(x, bias, T, y); torch.cuda.synchronize(); t1 = time.time()
    try:
        layer.check(); ok = "ok"
    except Exception as ex:
        ok = str(ex)[:80]
        ep = layer.read("restore_epoch").view(np.uint32)[0]
        print("epoch", ep, "layout", layer.read("layout", 0).reshape(E, N).tolist())
        for v in range(N):
            print(" rank", v, "ready[slot][src]", layer.read("ready", v).view(np.uint32).reshape(C, N).tolist())
    layer.backward(dy, dx); torch.cuda.synchronize(); t2 = time.time()
    print(os.environ.get("TAG"), i, f"fwd {1e3*(t1-t0):.1f} ms bwd {1e3*(t2-t1):.1f} ms", ok, flush=True)
layer.close()
