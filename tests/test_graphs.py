"""CUDA-graph capture of layer calls: after one plain call has
built and uploaded a plan's work list, multi_strategy_attention captures into
a CUDA graph (global capture mode: no uncaptured stream work is touched) and
the replay reproduces the direct calls bit for bit, Cached-head copies and
cache commits included. A plan never run before cannot be captured."""
import pytest
import torch

from paper_2503_22796_b200 import api
from paper_2503_22796_b200.api import UnsupportedError

pytestmark = pytest.mark.gpu


def _layer(H=6, NV=1024, NT=77, D=64, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    N = NV + NT
    dims = api.AttentionDims(H, D, NV, NT)
    q, k, v = (torch.randn(1, H, N, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    return dims, q, k, v


@pytest.mark.parametrize("D", [64, 128])
def test_captured_layers_replay_bitwise(D):
    dims, q, k, v = _layer(D=D)
    H, N = dims.n_heads, dims.seq_len()
    L = 3
    cache = api.HeadCache(L, H, N, D)
    plans = [api.LayerPlan.parse("F A0 C A2 C F"), api.LayerPlan.parse("C C A1 F A0 C"),
             api.LayerPlan.parse("A3 F F C A0 A1")]
    outs = [torch.empty_like(q) for _ in range(L)]
    for l in range(L):  # t = 0 fills the cache; t = 1 builds each plan's work list
        api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, l, 0, dims, 128, out=outs[l])
    for l in range(L):
        api.multi_strategy_attention(q, k, v, plans[l], cache, l, 1, dims, 128, out=outs[l])
    torch.cuda.synchronize()
    ref = [o.clone() for o in outs]
    slots = [[cache.fetch(l, h) for h in range(H)] for l in range(L)]

    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        for l in range(L):
            api.multi_strategy_attention(q, k, v, plans[l], cache, l, 1, dims, 128, out=outs[l])
    for o in outs:
        o.zero_()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    for l in range(L):
        assert torch.equal(outs[l], ref[l]), l
        for h in range(H):  # the commits replayed the same bits into the slots
            assert torch.equal(cache.fetch(l, h), slots[l][h]), (l, h)


@pytest.mark.filterwarnings("ignore:The CUDA Graph is empty")
def test_capturing_a_plan_never_run_is_refused():
    dims, q, k, v = _layer(seed=1)
    H = dims.n_heads
    cache = api.HeadCache(1, H, dims.seq_len(), dims.head_dim)
    out = torch.empty_like(q)
    api.multi_strategy_attention(q, k, v, api.LayerPlan.all_full(H), cache, 0, 0, dims, 128, out=out)
    torch.cuda.synchronize()
    fresh = api.LayerPlan.parse("A5 A5 C F A5 C")  # this work list was never built
    g = torch.cuda.CUDAGraph()
    with pytest.raises(UnsupportedError, match="plain call"):
        with torch.cuda.graph(g, stream=torch.cuda.Stream()):
            api.multi_strategy_attention(q, k, v, fresh, cache, 0, 1, dims, 128, out=out)
    torch.cuda.synchronize()
    # and after a plain call it captures
    api.multi_strategy_attention(q, k, v, fresh, cache, 0, 1, dims, 128, out=out)
    torch.cuda.synchronize()
    ref = out.clone()
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=torch.cuda.Stream()):
        api.multi_strategy_attention(q, k, v, fresh, cache, 0, 1, dims, 128, out=out)
    out.zero_()
    g2.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)

