"""Benchmark of the fused head-wise attention path (BASELINE.json metric):

  joint-attention layer latency & effective TFLOPS at FLUX 2K (16.9k tok),
  vs dense & CPU.

Workload (BASELINE.json configs[2]): one FLUX.1 2K joint-attention layer,
16384 image + 512 text tokens, 24 heads, d=128, bf16, mask block 128, the
paper's ~68% reduction plan "FLUX68" (6 Full, 8 Arrow(8), 4 Arrow(0),
6 Cached) at t=1 with every cache slot filled at t=0.
A step = one dfa2c_mha_forward call (ONE kernel launch) over one sample.

--gpus N: one process per GPU (this script re-launches itself under
torch.distributed.run when WORLD_SIZE is unset). `value` is the batch-
sharded layer (config 4's sharding: one FLUX sample per GPU, no data-path
collective; weak scaling). The same line carries `row_sharded`: ONE sample
split over the N GPUs by dfa2c_mha_forward_sharded (contiguous cost-
balanced row ranges, one fused launch per rank, NCCL all-gather in place)
— compute-only and compute + gather, strong scaling.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
PARITY_MAX_REL, PARITY_MAX_RSE = 1e-2, 5e-5  # DESIGN.md §4, SURVEY.md §8c


def dense_layer_flops() -> int:
    return H * 4 * D * N * N


def config():
    """Identical for both arms (the driver compares them)."""
    return {"workload": "FLUX.1 2K joint-attention layer (BASELINE configs[2])", "n_visual": NV, "n_text": NT,
            "heads": H, "head_dim": D, "mask_block": BLOCK, "plan": "FLUX68: " + PLAN, "samples_per_gpu": 1,
            "token_order": "visual_first",
            "l2": "no flush; per-step inputs q/k/v/out = 415 MB > 126 MB L2"}


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
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw,power.limit")

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
        sm, mx, reasons, watts, limit = [], None, set(), [], None
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
            try:  # board power: the sw_power_cap evidence
                watts.append(float(parts[6]))
                limit = float(parts[7])
            except (IndexError, ValueError):
                pass
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
               "samples": len(sm)}
        if watts:
            out["power_w"] = statistics.median(watts)
            out["power_limit_w"] = limit
        return out


def host_inputs(seed_base=0):
    """The step's inputs, generated once on the host (seeded, bf16): q/k/v
    [1, H, N, D] and the t=0 cache slots [H, N, D]. The GPU arm copies them
    to HBM; the CPU legs read the same values widened to f32."""
    import torch

    g = torch.Generator().manual_seed(seed_base + 1)
    q, k, v = (torch.randn(1, H, N, D, generator=g).to(torch.bfloat16) for _ in range(3))
    slots = torch.randn(H, N, D, generator=g).to(torch.bfloat16)
    return q, k, v, slots


def as_f32_numpy(x):
    import numpy as np

    return np.ascontiguousarray(x.float().numpy().reshape(H, N, D))


def cpu_layer(q, k, v, slots, threads=None, heads=None):
    """The reference's own CPU kernels (oracle/_ref, compiled from the
    unmodified /root/reference sources) over `heads` of the layer: Full ->
    dense_tiled_attention, Arrow(w) -> sparse_attention_forward (both
    parallel over query blocks), Cached -> copy; DFA2_THREADS = all host
    cores. q/k/v/slots: f32 numpy [H, N, D]. Returns (seconds, cores, out)."""
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
    return time.perf_counter() - t0, cores, out


def parity(gpu_out, ref_out):
    """Whole-layer parity of the GPU output against the reference CPU layer
    on the same inputs: per head max|gpu-ref|/max|ref| and RSE (the
    reference's rse, src/calibrate.cpp:18-87, in f64); Cached heads bitwise."""
    import numpy as np

    g = gpu_out.float().cpu().numpy().reshape(H, N, D).astype(np.float64)
    kinds = [s for s in PLAN.split()]
    rels, rses, cached_equal = [], [], True
    for h in range(H):
        r = ref_out[h].astype(np.float64)
        e = g[h] - r
        rels.append(float(np.abs(e).max() / np.abs(r).max()))
        den = float(((r - r.mean()) ** 2).sum())
        rses.append(float((e ** 2).sum() / den))
        if kinds[h] == "C":
            cached_equal &= bool(np.array_equal(g[h], r))
    worst = int(np.argmax(rels))
    ok = max(rels) <= PARITY_MAX_REL and max(rses) <= PARITY_MAX_RSE and cached_equal
    return {"checked": f"all {H} heads x {N} rows x {D} cols vs the reference CPU layer (oracle/_ref) on the same "
                       "bf16 inputs",
            "max_rel": max(rels), "rse_per_head_max": max(rses), "worst_head": worst,
            "worst_head_kind": kinds[worst], "cached_heads_bitwise": cached_equal,
            "tolerance": {"max_rel": PARITY_MAX_REL, "rse": PARITY_MAX_RSE}, "pass": ok}


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
    q, k, v, slots = (as_f32_numpy(x) for x in host_inputs())
    first, _, _ = cpu_layer(q, k, v, slots)
    heads = CPU_SAMPLE_HEADS if first * (args.steps + args.warmup) <= 150.0 else CPU_SAMPLE_HEADS[:8]
    for _ in range(args.warmup - 1):
        cpu_layer(q, k, v, slots, heads=heads)
    times = []
    cores = 1
    for _ in range(args.steps):
        dt, cores, _ = cpu_layer(q, k, v, slots, heads=heads)
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
            "config": config(), "layer_ms": sec * 1e3 * H / len(heads),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def spawn(args):
    """--gpus N without a torchrun environment: relaunch under
    torch.distributed.run, one process per GPU, and pass its exit code on."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have}", file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def cpp_f32_dropin():
    """The reference's calling convention end to end: dfa2::multi_strategy_attention
    with host f32 Tensors (tools/cpp_api_bench, built by __graft_entry__.build())."""
    exe = os.path.join(ROOT, "tools", "cpp_api_bench_bin")
    if not os.path.exists(exe):
        return {"unavailable": "tools/cpp_api_bench_bin not built"}
    try:
        r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
        rec = json.loads(r.stdout.strip().splitlines()[-1])
        ms = rec["ms_per_call"]
        return {"value": dense_layer_flops() / (ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ms,
                "h2d_bytes_per_step": 3 * 18 * N * D * 4, "d2h_bytes_per_step": H * N * D * 4,
                "api": rec["api"] + " (f32 host in/out; bf16 over PCIe, rounding on host)"}
    except Exception as e:  # a reported figure, never the product
        return {"unavailable": str(e)[:200]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline / parity leg")
    ap.add_argument("--ncu", action="store_true", help="short run for profiler captures (no e2e/cpu legs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)

    import torch
    import torch.distributed as dist

    from paper_2503_22796_b200 import api

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
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
    hq, hk, hv, hslots = host_inputs(1000 * rank)  # this rank's own sample
    q, k, v = (x.cuda() for x in (hq, hk, hv))
    out = torch.empty_like(q)
    cache = api.HeadCache(1, H, N, D, batch=1)
    slots = hslots.cuda()
    for h in range(H):  # t = 0: every slot produced
        cache.store(0, h, slots[h], 0)
    lp = api.LayerPlan.parse(PLAN)
    full = api.LayerPlan.all_full(H)
    plan_fl = api.plan_flops(lp, dims, BLOCK)
    stream = torch.cuda.current_stream()

    def step(plan, t=1):
        api.multi_strategy_attention(q, k, v, plan, cache, 0, t, dims, BLOCK, out=out)

    def timed(fn, steps, warmup, min_warm_s=0.0):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < min_warm_s:  # keep clocks at load for the sampler
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        l0 = api.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1) / steps
        return max_over_ranks(ms), api.launch_count() - l0

    # headline: FLUX68 layer, inputs resident in HBM
    with ClockSampler(local) as clk:
        ms, launches = timed(lambda: step(lp), args.steps, args.warmup, min_warm_s=0.0 if args.ncu else 1.0)
        time.sleep(0.25)
    clocks = clk.summary()
    gpu_out = out.clone()  # the FLUX68 layer output of this rank's sample (for the parity leg)
    # dense comparison through the same kernel (all-Full plan; no cached heads)
    dense_ms, _ = timed(lambda: step(full), max(3, args.steps // 2), 2)

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
            "config": config(), "parallelism": f"batch-sharded x{world} (one FLUX 2K sample per GPU)",
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
        # ONE sample over the `world` GPUs (strong scaling): contiguous
        # cost-balanced row ranges, one fused launch per rank, in-place NCCL
        # all-gather + cache completion (dfa2c_mha_forward_sharded).
        comm = api.NcclComm.create(rank, world) if world > 1 else None
        sq, sk, sv = (x.cuda() for x in host_inputs(0)[:3])  # the same sample on every rank
        s_out = torch.empty_like(sq)
        s_cache = api.HeadCache(1, H, N, D, batch=1)
        for h in range(H):
            s_cache.store(0, h, slots[h], 0)
        bounds = api.shard_rows(lp, dims, BLOCK, world)

        def sharded(c):
            api.multi_strategy_attention_sharded(sq, sk, sv, lp, s_cache, 0, 1, dims, BLOCK, rank, world, comm=c,
                                                 out=s_out)

        s_compute, _ = timed(lambda: sharded(None), args.steps, args.warmup)
        s_layer, _ = timed(lambda: sharded(comm), args.steps, args.warmup) if world > 1 else (s_compute, 0)
        p2p = None
        if world > 1:
            # the same layer assembled over peer memory: each rank's kernel
            # stores its rows into every rank's buffer (CUDA IPC over
            # NVLink), no collective; a step ends when every rank's launch
            # has completed (device sync + barrier inside the timed region)
            from paper_2503_22796_b200 import parallel

            peers = parallel.PeerOutputs(s_out, rank, world)

            def p2p_step():
                api.multi_strategy_attention_sharded_p2p(sq, sk, sv, lp, s_cache, 0, 1, dims, BLOCK, rank, world,
                                                         peers.outs)
                torch.cuda.synchronize()
                barrier()

            p2p_ms, _ = timed(p2p_step, args.steps, args.warmup)
            barrier()
            peers.close()
            p2p = {"layer_ms": p2p_ms, "value": dense_fl / (p2p_ms * 1e-3) / 1e12, "unit": UNIT,
                   "how": "dfa2c_mha_forward_sharded_p2p: output boxes stored to every rank's buffer from the "
                          "kernel epilogue (CUDA IPC / NVLink), no NCCL; includes a device sync + barrier per step"}
        line["row_sharded"] = {
            "what": "one FLUX68 sample split over the GPUs (dfa2c_mha_forward_sharded): strong scaling",
            "n_gpus": world, "compute_ms": s_compute, "layer_ms": s_layer,
            "gather": "NCCL group of W in-place broadcasts (all-gather-v) + cache completion" if world > 1 else None,
            "value": dense_fl / (s_layer * 1e-3) / 1e12, "unit": UNIT,
            "rows_per_rank": [int(bounds[r + 1] - bounds[r]) for r in range(world)],
            "nccl_ranks": world if comm is not None else 0, "p2p_assembly": p2p}
        if comm is not None:
            comm.close()
        if world == 1:
            # strong scaling emulated on this GPU: each rank r of W runs exactly
            # the launch its own GPU would (same row range, no gather), timed
            # alone; the per-GPU compute at W GPUs is the max over ranks
            emu = {}
            for W in (2, 4, 8):
                per, per_p2p = [], []
                bufs = [s_out] + [torch.empty_like(s_out) for _ in range(W - 1)]
                for r in range(W):
                    fn = lambda: api.multi_strategy_attention_sharded(sq, sk, sv, lp, s_cache, 0, 1, dims, BLOCK,
                                                                      r, W, out=s_out)
                    per.append(timed(fn, max(5, args.steps // 2), 3)[0])
                    # the peer-memory variant: every output box also stored to the W-1 other
                    # ranks' buffers (here on this GPU's HBM instead of NVLink)
                    extra = iter(bufs[1:])
                    outs = [s_out if j == r else next(extra) for j in range(W)]  # outs[r]: this rank's own
                    fp = lambda: api.multi_strategy_attention_sharded_p2p(sq, sk, sv, lp, s_cache, 0, 1, dims,
                                                                          BLOCK, r, W, outs)
                    per_p2p.append(timed(fp, max(5, args.steps // 2), 3)[0])
                del bufs
                emu[str(W)] = {"per_rank_compute_ms": per, "max_ms": max(per),
                               "x_ideal_vs_1gpu_layer": max(per) * W / ms,
                               "p2p_per_rank_ms": per_p2p, "p2p_max_ms": max(per_p2p)}
            line["row_sharded"]["emulated_ranks"] = {
                "what": "per-GPU compute of the row-sharded layer at W GPUs, every rank's launch timed alone on "
                        "this GPU (gather not included); x_ideal_vs_1gpu_layer = max_ms * W / layer_ms",
                "worlds": emu}

        # e2e through the public API with HOST buffers: dfa2c_mha_forward_host
        # uploads the computed heads' q/k/v from pinned memory in head groups,
        # runs each group's fused launch as its inputs land, and downloads
        # outputs (cached heads straight from their slots) — all inside the
        # timed region, every step.
        pq, pk, pv = (x.pin_memory() for x in (hq, hk, hv))
        ho = torch.empty(q.shape, dtype=torch.bfloat16).pin_memory()

        def e2e_step():
            api.multi_strategy_attention_host(pq, pk, pv, lp, cache, 0, 1, dims, BLOCK, out=ho)

        for _ in range(2):
            e2e_step()
        step(lp)
        torch.cuda.synchronize()
        if not torch.equal(ho.to("cuda"), out):  # same plan, inputs and cache: bitwise the device-path output
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
        line["e2e_cpp_f32"] = cpp_f32_dropin()
        try:
            cq, ck, cv, cs = (as_f32_numpy(x) for x in (hq, hk, hv, hslots))
            # whole layers until ~10 s of CPU work (at least one)
            secs, ref_out = [], None
            while not secs or (sum(secs) < 10.0 and len(secs) < 5):
                sec, cores, ref_out = cpu_layer(cq, ck, cv, cs)
                secs.append(sec)
            sec = sum(secs) / len(secs)
            sample_flops = len(CPU_SAMPLE_HEADS) * 4 * D * N * N
            line["cpu_baseline"] = {
                "value": sample_flops / sec / 1e12, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"the whole FLUX68 layer ({len(CPU_SAMPLE_HEADS)} heads) x {len(secs)} through oracle/_ref "
                          f"(reference dense_tiled / sparse_attention_forward, DFA2_THREADS={cores}); "
                          f"{sec:.2f} s per layer, {sum(secs):.1f} s total"}
            line["parity"] = parity(gpu_out, ref_out)
        except Exception as e:  # the CPU leg is a reported baseline, never the product
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
