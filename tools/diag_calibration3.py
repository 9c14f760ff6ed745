import cProfile, pstats, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2503_22796_b200 import api
L, H, nv, nt, d, B, T = 57, 24, 16384, 512, 128, 128, 2
n = nv + nt
dims = api.AttentionDims(H, d, nv, nt)
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
qs = [q, (q.float() + 0.05 * torch.randn(H, n, d, device="cuda", generator=g)).to(torch.bfloat16)]
cfg = api.CalibrationConfig(api.make_candidates([0, 2, 8, 16, 32], include_cached=True), 0.4, 1.5)
for rep in range(4):
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    r = api.calibrate_model(lambda t, l: qs[t], lambda t, l: k, lambda t, l: v, dims, T, L, B, cfg)
    torch.cuda.synchronize()
    pr.disable()
    dt = (time.perf_counter() - t0) / (T * L) * 1e3
    print(f"rep {rep}: {dt:.2f} ms/layer", flush=True)
    if dt > 15:
        pstats.Stats(pr).sort_stats("tottime").print_stats(8)
    del r
