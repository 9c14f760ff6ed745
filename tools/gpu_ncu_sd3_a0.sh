cat > /tmp/sd3_once.py <<'PY'
import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2503_22796_b200 import api
H, nv, nt, d, B = 24, 4096, 333, 64, 128
n = nv + nt
dims = api.AttentionDims(H, d, nv, nt)
q, k, v = (torch.randn(1, H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
lp = api.LayerPlan.parse(" ".join([sys.argv[1]] * H))
for _ in range(4):
    api.multi_strategy_attention(q, k, v, lp, None, 0, 0, dims, B, out=out)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/prof_sd3v3_A0 -f python /tmp/sd3_once.py A0 > gpurun_out/ncu_sd3v3.log 2>&1
tail -1 gpurun_out/ncu_sd3v3.log
