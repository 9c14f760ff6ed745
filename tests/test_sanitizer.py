"""compute-sanitizer (memcheck, racecheck, synccheck) over small layers of
every kernel path: d = 64 and 128, Full / Arrow / Cached items with cache
commits, split-KV chunks and their combine, the fused calibration pass, a
mask block other than the tile (element masking), text rows halved across
the two lanes, row-sharded launches (unequal key chunks) and the SIMT path
for head_dim > 128."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import sys; sys.path.insert(0, %r)
import torch
from paper_2503_22796_b200 import api
for d in (64, 128):
    H, nv, nt, B = 4, 1024, 77, 128
    n = nv + nt
    dims = api.AttentionDims(H, d, nv, nt)
    q, k, v = (torch.randn(H, n, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    cache = api.HeadCache(1, H, n, d)
    api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, 0, 0, dims, B)
    api.multi_strategy_attention(q, k, v, api.LayerPlan.parse("F A0 A2 C"), cache, 0, 1, dims, B)
    api.set_split_kv(True)
    api.multi_strategy_attention(q, k, v, api.LayerPlan.parse("A0 A1 C C"), cache, 0, 2, dims, B)
    api.set_split_kv(False)
    api.influence_for_layer(q, k, v, api.make_candidates([0, 2], True), cache, 0, 3, dims, B)
    api.multi_strategy_attention(q, k, v, api.LayerPlan.parse("F A0 A2 C"), cache, 0, 4, dims, 64)
# text rows halved across the lanes (d = 64, narrow windows)
dims = api.AttentionDims(2, 64, 4096, 333)
q, k, v = (torch.randn(2, 4429, 64, device="cuda").to(torch.bfloat16) for _ in range(3))
api.multi_strategy_attention(q, k, v, api.LayerPlan.parse("A0 A1"), None, 0, 0, dims, 128)
# row-sharded launches (unequal key chunks and their combine), ranks of 2 and 4
dims = api.AttentionDims(4, 128, 1024, 77)
q, k, v = (torch.randn(4, 1101, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
cache = api.HeadCache(1, 4, 1101, 128)
api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(4), cache, 0, 0, dims, 128)
for world in (2, 4):
    for rank in range(world):
        api.multi_strategy_attention_sharded(q, k, v, api.LayerPlan.parse("F A0 C A2"), cache, 0, 1, dims, 128,
                                             rank, world)
# head_dim > 128 (SIMT path)
dims = api.AttentionDims(2, 160, 200, 40)
q, k, v = (torch.randn(2, 240, 160, device="cuda").to(torch.bfloat16) for _ in range(3))
api.multi_strategy_attention(q, k, v, api.LayerPlan.parse("F A0"), None, 0, 0, dims, 64)
torch.cuda.synchronize()
print("case ok")
''' % ROOT


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and os.path.exists(p):
            return p
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_kernels_are_sanitizer_clean(tool, tmp_path):
    case = tmp_path / "case.py"
    case.write_text(CASE)
    r = subprocess.run([_sanitizer(), "--tool", tool, "--error-exitcode", "99", sys.executable, str(case)],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "case ok" in out, out[-3000:]
    assert ("0 errors" in out) or ("0 hazards" in out), out[-3000:]
