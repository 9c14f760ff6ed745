"""Benchmark of the fused head-wise attention path (BASELINE.json metric):

  joint-attention layer latency & effective TFLOPS at FLUX 2K (16.9k tok),
  vs dense & CPU.

Workload (BASELINE.json configs[2]): one FLUX.1 2K joint-attention layer,
16384 image + 512 text tokens, 24 heads, d=128, bf16, mask block 128, the
paper's ~68% reduction plan "FLUX68" (6 Full, 8 Arrow(8), 4 Arrow(0),
6 Cached) at t=1 with every cache slot filled at t=0.
A step = one dfa2c_mha_forward call (ONE kernel launch) over one sample.
With --gpus N (torchrun, one process per GPU) each rank runs its own sample
(batch/sample sharding, no data-path collective): weak scaling.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "joint-attention layer latency & effective TFLOPS at FLUX 2K (16.9k tok), vs dense & CPU"
UNIT = "TFLOPS (dense-equivalent: H*4*d*N^2 / layer time)"
H, NV, NT, D, BLOCK = 24, 16384, 512, 128, 128
N = NV + NT
PLAN = "F A8 C A0 F A8 C A8 F A8 C A0 F A8 C A0 F A8 C A8 F A8 C A0"
CPU_SAMPLE_HEADS = list(range(H))  # the whole FLUX68 layer (6 F, 8 A8, 4 A0, 6 C): no extrapolation


def dense_layer_flops() -> int:
    return H * 4 * D * N * N


def config(extra=None):
    c = {"workload": "FLUX.1 2K joint-attention layer (BASELINE configs[2])", "n_visual": NV, "n_text": NT,
         "heads": H, "head_dim": D, "mask_block": BLOCK, "plan": "FLUX68: " + PLAN, "samples_per_gpu": 1,
         "token_order": "visual_first",
         "l2": "no flush; per-step inputs q/k/v/out = 415 MB > 126 MB L2"}
    if extra:
        c.update(extra)
    return c


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), \
            float(p["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_layer_sample(q, k, v, slots, threads=None, heads=None):
    """The reference's own CPU kernels (oracle/_ref, compiled from
    /root/reference sources) on heads CPU_SAMPLE_HEADS of the same layer:
    Full -> dense_tiled_attention, Arrow(w) -> sparse_attention_forward,
    Cached -> copy; DFA2_THREADS = all host cores. Returns (seconds, cores)."""
    import numpy as np

    import oracle
    from oracle import c_float, c_int32, c_int64, ptr

    cores = threads or os.cpu_count() or 1
    os.environ["DFA2_THREADS"] = str(cores)
    from paper_2503_22796_b200 import api

    lp = api.LayerPlan.parse(PLAN)
    kinds = np.array([api._KIND_CODE[s.kind] for s in lp.strategies], np.int32)
    wins = np.array([s.window_blocks for s in lp.strategies], np.int64)
    heads = np.array(CPU_SAMPLE_HEADS if heads is None else heads, np.int64)
    out = np.zeros_like(q)
    t0 = time.perf_counter()
    oracle.ref_check(oracle.ref().ref_layer_sample(ptr(q, c_float), ptr(k, c_float), ptr(v, c_float),
                                                   ptr(slots, c_float), ptr(out, c_float), H, D, NV, NT, 0, BLOCK,
                                                   ptr(kinds, c_int32), ptr(wins, c_int64), ptr(heads, c_int64),
                                                   len(heads)))
    return time.perf_counter() - t0, cores


def host_sample_inputs(seed_base=0):
    """bf16-rounded f32 copies of the bench inputs for the CPU sample (only
    the sampled heads are materialised; others stay zero and are not read)."""
    import numpy as np
    import torch

    def gen(seed, heads):
        g = torch.Generator().manual_seed(seed)
        x = torch.zeros(H, N, D, dtype=torch.float32)
        full = torch.randn(len(heads), N, D, generator=g).to(torch.bfloat16).float()
        for i, h in enumerate(heads):
            x[h] = full[i]
        return np.ascontiguousarray(x.numpy())

    hs = CPU_SAMPLE_HEADS
    return gen(seed_base + 1, hs), gen(seed_base + 2, hs), gen(seed_base + 3, hs), gen(seed_base + 100, hs)


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path
    (oracle/_ref) on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    if not oracle.ref_available():
        try:
            oracle.build(ref=True)
        except Exception:
            pass
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdfa2ref.so not built"}))
        return
    # A step is the whole layer. If the first (warm-up) layer shows that
    # K + W whole-layer steps would exceed ~150 s, each step samples the
    # first 8 heads (F A8 C A0 F A8 C A8) instead, keeping the run within a
    # few minutes.
    q, k, v, slots = host_sample_inputs()
    first, _ = cpu_layer_sample(q, k, v, slots)
    heads = CPU_SAMPLE_HEADS if first * (args.steps + args.warmup) <= 150.0 else CPU_SAMPLE_HEADS[:8]
    for _ in range(args.warmup - 1):
        cpu_layer_sample(q, k, v, slots, heads=heads)
    times = []
    cores = 1
    for _ in range(args.steps):
        dt, cores = cpu_layer_sample(q, k, v, slots, heads=heads)
        times.append(dt)
    sec = sum(times) / len(times)
    sample_flops = len(heads) * 4 * D * N * N
    value = sample_flops / sec / 1e12
    sample = (f"{'the whole FLUX68 layer' if len(heads) == H else f'heads {heads} of the FLUX68 layer'} per step "
              f"({len(heads)} heads, full N); Full via the reference's dense_tiled_attention, Arrow via "
              "sparse_attention_forward (parallel over query blocks), Cached via copy; "
              "value = dense-equivalent FLOPs of those heads / time")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded N(0,1), bf16-rounded)",
            "config": config({"cpu_sample": "whole layer"}),
            "layer_ms": sec * 1e3 * H / len(heads),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_head_mode(args, rank, world, barrier, max_over_ranks):
    """One FLUX sample on `world` GPUs: heads LPT-sharded by plan cost, one
    fused launch per rank over the full plan with the other ranks' heads
    DFA2C_SKIP, NCCL all-gather of the bf16 output heads
    (paper_2503_22796_b200.parallel). Strong scaling."""
    import torch

    from paper_2503_22796_b200 import api, parallel

    dims = api.AttentionDims(H, D, NV, NT)
    lp = api.LayerPlan.parse(PLAN)
    shard = parallel.make_head_shard(lp, dims, BLOCK, world, rank)
    gen = torch.Generator(device="cuda")

    def randn(seed, *shape):
        gen.manual_seed(seed)
        return torch.randn(*shape, device="cuda", dtype=torch.float32, generator=gen).to(torch.bfloat16)

    q, k, v = (randn(s, H, N, D) for s in (1, 2, 3))  # the same sample on every rank
    nh = len(shard.heads)
    cache = api.HeadCache(1, H, N, D)  # layer-shaped; only this rank's slots are touched
    for h in shard.heads:
        cache.store(0, h, randn(100 + h, N, D), 0)
    full = torch.empty_like(q)
    skip = [h for h in range(H) if h not in set(shard.heads)]
    stream = torch.cuda.current_stream()

    def compute():  # one fused launch over the full plan, other ranks' heads DFA2C_SKIP
        if nh:
            api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, BLOCK, out=full, skip_heads=skip)

    idx = torch.tensor(shard.heads, device="cuda", dtype=torch.long)

    def step():
        compute()
        parallel.gather_heads(full.index_select(0, idx), shard, full)

    # compute + gather overlapped per head group (parallel.pipelined_sharded_attention)
    n_groups = args.head_groups or (3 if nh >= 12 else 2 if nh >= 6 else 1)
    comm = torch.cuda.Stream()

    def compute_group(hs):
        owned = set(hs)
        api.multi_strategy_attention(q, k, v, lp, cache, 0, 1, dims, BLOCK, out=full,
                                     skip_heads=[h for h in range(H) if h not in owned])

    def piped():
        parallel.pipelined_sharded_attention(compute_group, full, shard, n_groups, comm_stream=comm)

    def timed(fn, steps):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / steps)

    compute_ms = timed(compute, args.steps)
    serial_ms = timed(step, args.steps)
    piped_ms = timed(piped, args.steps)
    ms = min(serial_ms, piped_ms)
    dense_fl = dense_layer_flops()
    line = {"metric": METRIC, "value": dense_fl / (ms * 1e-3) / 1e12, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) bf16)",
            "config": config({"parallelism": f"head-sharded x{world} (LPT on plan cost) + NCCL all-gather"}),
            "layer_ms": ms, "compute_only_ms": compute_ms, "compute_then_gather_ms": serial_ms,
            "overlapped_ms": piped_ms, "head_groups": n_groups,
            "heads_per_rank": [len(o) for o in shard.all_heads]}
    if rank == 0:
        print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--ncu", action="store_true", help="short run for profiler captures (no e2e/cpu legs)")
    ap.add_argument("--head-groups", type=int, default=0,
                    help="--mode head: head groups whose gather overlaps the next group's compute (0 = auto)")
    ap.add_argument("--mode", default="sample", choices=["sample", "head"],
                    help="sample: one FLUX sample per GPU (weak scaling, no collective); "
                         "head: one sample split over the GPUs by LPT head sharding + NCCL all-gather (strong)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2503_22796_b200 import api

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    dims = api.AttentionDims(H, D, NV, NT)
    if args.mode == "head":
        return run_head_mode(args, rank, world, barrier, max_over_ranks)
    seed0 = 1000 * rank
    gen = torch.Generator(device="cuda")

    def randn(seed, *shape):
        gen.manual_seed(seed)
        return torch.randn(*shape, device="cuda", dtype=torch.float32, generator=gen).to(torch.bfloat16)

    q = randn(seed0 + 1, 1, H, N, D)
    k = randn(seed0 + 2, 1, H, N, D)
    v = randn(seed0 + 3, 1, H, N, D)
    out = torch.empty_like(q)
    cache = api.HeadCache(1, H, N, D, batch=1)
    for h in range(H):  # t = 0: every slot produced
        cache.store(0, h, randn(seed0 + 100 + h, N, D), 0)
    lp = api.LayerPlan.parse(PLAN)
    full = api.LayerPlan.all_full(H)
    plan_fl = api.plan_flops(lp, dims, BLOCK)
    stream = torch.cuda.current_stream()

    def step(plan, t=1):
        api.multi_strategy_attention(q, k, v, plan, cache, 0, t, dims, BLOCK, out=out)

    def timed(plan, steps, warmup, min_warm_s=0.0):
        for _ in range(warmup):
            step(plan)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < min_warm_s:  # keep clocks at load for the sampler
            for _ in range(20):
                step(plan)
            torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        l0 = api.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step(plan)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1) / steps
        return max_over_ranks(ms), api.launch_count() - l0

    # headline: FLUX68 layer, inputs resident in HBM
    with ClockSampler(local) as clk:
        ms, launches = timed(lp, args.steps, args.warmup, min_warm_s=0.0 if args.ncu else 1.0)
        time.sleep(0.25)
    clocks = clk.summary()
    # dense comparison through the same kernel (all-Full plan; no cached heads)
    dense_ms, _ = timed(full, max(3, args.steps // 2), 2)

    dense_fl = dense_layer_flops()
    value = world * dense_fl / (ms * 1e-3) / 1e12
    peak_burst, peak_sust, hbm, src = peaks()
    achieved = plan_fl / (ms * 1e-3) / 1e12  # one kernel launch per step: step == kernel duration
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_latest.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded N(0,1) bf16; random cache slots)",
            "config": config({"parallelism": f"sample-sharded x{world} (one FLUX 2K sample per GPU)"}),
            "layer_ms": ms, "dense_ms": dense_ms, "speedup_vs_dense": dense_ms / ms,
            "plan_flops": plan_fl, "dense_flops": dense_fl, "flop_reduction": 1 - plan_fl / dense_fl,
            "computed_tflops": achieved, "dense_path_tflops": dense_fl / (dense_ms * 1e-3) / 1e12,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_burst, "unit": "TFLOP/s",
                         "frac": achieved / peak_burst, "traffic": traffic,
                         "peak_source": f"{src} bf16_tflops (burst); sustained {peak_sust}",
                         "frac_of_sustained": achieved / peak_sust, "kernel": "attn_fwd_sm100<128>",
                         "algorithmic": "plan_flops = sum over non-cached heads of 4*d*active_positions"},
            "gpu_launches": launches, "clocks": clocks}

    if not args.ncu:
        # e2e through the public API with HOST buffers: dfa2c_mha_forward_host
        # uploads the computed heads' q/k/v from pinned memory in head groups,
        # runs each group's fused launch as its inputs land, and downloads
        # outputs (cached heads straight from their slots) — all inside the
        # timed region, every step.
        hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
        ho = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()

        def e2e_step():
            api.multi_strategy_attention_host(hq, hk, hv, lp, cache, 0, 1, dims, BLOCK, out=ho)

        for _ in range(2):
            e2e_step()
        step(lp)
        torch.cuda.synchronize()
        if not torch.equal(ho.to("cuda"), out):  # same plan, same inputs: bitwise the device-path output
            raise RuntimeError("host-buffer path disagrees with the device path")
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ke = max(3, min(args.steps, 10))
        e0.record(stream)
        for _ in range(ke):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / ke)
        head_bytes = N * D * 2
        n_comp = sum(1 for s_ in lp.strategies if s_.kind != "cached")
        line["e2e"] = {"value": world * dense_fl / (e2e_ms * 1e-3) / 1e12, "unit": UNIT,
                       "h2d_bytes_per_step": 3 * n_comp * head_bytes, "d2h_bytes_per_step": H * head_bytes,
                       "ms_per_step": e2e_ms,
                       "api": "paper_2503_22796_b200.api.multi_strategy_attention_host -> dfa2c_mha_forward_host "
                              "(pinned host q/k/v in, host out; only computed heads' q/k/v uploaded)"}

    if rank == 0 and world == 1 and not args.no_cpu and not args.ncu:
        try:
            hq_, hk_, hv_, hs_ = host_sample_inputs()
            # whole layers until ~10 s of CPU work (at least one)
            secs = []
            while not secs or (sum(secs) < 10.0 and len(secs) < 5):
                sec, cores = cpu_layer_sample(hq_, hk_, hv_, hs_)
                secs.append(sec)
            sec = sum(secs) / len(secs)
            sample_flops = len(CPU_SAMPLE_HEADS) * 4 * D * N * N
            line["cpu_baseline"] = {
                "value": sample_flops / sec / 1e12, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"the whole FLUX68 layer ({len(CPU_SAMPLE_HEADS)} heads) x {len(secs)} through oracle/_ref "
                          f"(reference dense_tiled / sparse_attention_forward, DFA2_THREADS={cores}); "
                          f"{sec:.2f} s per layer, {sum(secs):.1f} s total"}
        except Exception as e:  # the CPU leg is a reported baseline, never the product
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
