"""Generates the golden vectors in tests/golden/ from the REFERENCE ITSELF.

Run in the container that has /root/reference (the build recipe compiles the
unmodified reference sources in place into oracle/_ref/libdfa2ref.so):

    make -C oracle all ref && python tests/golden/gen_golden.py

Every value below comes from a reference entry point through
oracle/ref_capi.cpp (build_arrow_mask, BlockMask stats, plan_flops,
sparse_attention_forward, attention_reference<double>, rse,
multi_strategy_attention + HeadCache, generate). Inputs are seeded numpy
gaussians (PCG64, reproducible anywhere) so only outputs are stored.
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402
from oracle import c_double, c_float, c_int32, c_int64, c_uint8, ptr, ref, ref_check  # noqa: E402

# (n_visual, n_text, order, B, w): the reference tests' geometries
# (tests/test_arrow.cpp:53-152, test_bench.cpp:21-32) plus the survey configs.
MASK_CASES = [
    (512, 128, 0, 128, 0), (512, 128, 0, 128, 3), (512, 128, 0, 128, 4), (512, 128, 0, 128, 100),
    (512, 0, 0, 128, 0), (512, 128, 1, 128, 0), (4 * 32, 0, 0, 32, 0), (260, 30, 0, 32, 9),
    (4096, 512, 0, 128, 0), (4096, 512, 0, 128, 6), (4096, 512, 0, 128, 13),
    (1024, 77, 0, 128, 0), (1024, 77, 0, 128, 2), (1024, 77, 0, 64, 0), (1024, 77, 0, 64, 2),
    (4096, 333, 0, 128, 0), (4096, 333, 1, 128, 0), (4096, 333, 0, 128, 8), (4096, 333, 0, 128, 31),
    (16384, 512, 0, 128, 0), (16384, 512, 0, 128, 8), (16384, 512, 1, 128, 8), (16384, 512, 0, 128, 64),
    (16384, 512, 0, 64, 16), (17, 0, 0, 8, 0), (120, 10, 0, 16, 1), (80, 16, 0, 16, 1), (40, 8, 0, 8, 0),
]
# plus 20 seeded random geometries like tests/test_arrow.cpp:98-110
_rng = np.random.default_rng(13)
for _ in range(20):
    MASK_CASES.append((int(1 + _rng.integers(300)), int(_rng.integers(60)), int(_rng.integers(2)),
                       int(1 + _rng.integers(48)), int(_rng.integers(5))))


def ref_mask(nv, nt, order, B, w):
    nb = c_int64()
    ref_check(ref().ref_arrow_mask(1, 8, nv, nt, order, B, w, None, ctypes.byref(nb)))
    m = np.zeros(nb.value * nb.value, np.uint8)
    ref_check(ref().ref_arrow_mask(1, 8, nv, nt, order, B, w, ptr(m, c_uint8), ctypes.byref(nb)))
    return m


def main():
    out = {}
    # --- masks + stats
    for i, (nv, nt, order, B, w) in enumerate(MASK_CASES):
        m = ref_mask(nv, nt, order, B, w)
        ap, fl, sp = c_int64(), c_int64(), c_double()
        ref_check(ref().ref_mask_stats(ptr(m, c_uint8), nv + nt, B, 64, ctypes.byref(ap), ctypes.byref(fl),
                                       ctypes.byref(sp)))
        out[f"mask{i}_geom"] = np.array([nv, nt, order, B, w], np.int64)
        out[f"mask{i}_bits"] = np.packbits(m)
        out[f"mask{i}_nbits"] = np.array([m.size], np.int64)
        out[f"mask{i}_stats"] = np.array([ap.value, fl.value], np.int64)
        out[f"mask{i}_sparsity"] = np.array([sp.value], np.float64)
    out["n_mask_cases"] = np.array([len(MASK_CASES)], np.int64)

    # --- plan_flops (dispatch.cpp:93-120)
    plans = {
        "cfg1": ((4, 64, 1024, 77, 0, 128), [0, 1, 1, 2], [0, 0, 2, 0]),
        "cfg1_b64": ((4, 64, 1024, 77, 0, 64), [0, 1, 1, 2], [0, 0, 2, 0]),
        "flux68": ((24, 128, 16384, 512, 0, 128),
                   [0, 1, 2, 1] * 6, sum(([0, 8, 0, 0 if g % 3 != 1 else 8] for g in range(6)), [])),
        "sd3_flux68": ((24, 64, 4096, 333, 0, 128),
                       [0, 1, 2, 1] * 6, sum(([0, 8, 0, 0 if g % 3 != 1 else 8] for g in range(6)), [])),
    }
    for name, ((H, d, nv, nt, order, B), kinds, wins) in plans.items():
        k = np.array(kinds, np.int32)
        w = np.array(wins, np.int64)
        f = c_int64()
        ref_check(ref().ref_plan_flops(H, d, nv, nt, order, B, ptr(k, c_int32), ptr(w, c_int64), ctypes.byref(f)))
        out[f"plan_{name}"] = np.array([H, d, nv, nt, order, B, f.value], np.int64)
        out[f"plan_{name}_kinds"] = k
        out[f"plan_{name}_windows"] = w

    # --- sparse forward (f32) and f64 oracle, small cases (test_arrow.cpp:154-236)
    att = [(256, 32, 32, 32, 0), (256, 32, 32, 32, 2), (14, 3, 8, 8, 0), (110, 20, 8, 16, 2), (256, 44, 64, 64, 1),
           (256, 44, 64, 48, 0), (200, 100, 128, 128, 0)]
    for i, (nv, nt, d, B, w) in enumerate(att):
        n = nv + nt
        q = oracle.gaussian((n, d), 1000 + 3 * i)
        k = oracle.gaussian((n, d), 1001 + 3 * i)
        v = oracle.gaussian((n, d), 1002 + 3 * i)
        m = ref_mask(nv, nt, 0, B, w)
        o32 = np.zeros((n, d), np.float32)
        ref_check(ref().ref_sparse_attention_forward(ptr(q, c_float), ptr(k, c_float), ptr(v, c_float),
                                                     ptr(o32, c_float), n, d, ptr(m, c_uint8), B, 0))
        q64, k64, v64 = (x.astype(np.float64) for x in (q, k, v))
        o64 = np.zeros((n, d), np.float64)
        ref_check(ref().ref_attention_reference_f64(ptr(q64, c_double), ptr(k64, c_double), ptr(v64, c_double),
                                                    ptr(o64, c_double), 1, n, d, ptr(m, c_uint8), B))
        out[f"att{i}_geom"] = np.array([nv, nt, d, B, w, 1000 + 3 * i], np.int64)
        out[f"att{i}_sparse_f32"] = o32
        out[f"att{i}_ref_f64"] = o64
    out["n_att_cases"] = np.array([len(att)], np.int64)

    # --- rse (calibrate.cpp:75-87)
    rs = []
    for i, n in enumerate([2, 16, 1000, 4096 * 8]):
        a = oracle.gaussian((n,), 500 + i)
        b = oracle.gaussian((n,), 600 + i) * 0.1 + a
        for mode in (0, 1):
            r = c_double()
            ref_check(ref().ref_rse(ptr(b, c_float), ptr(a, c_float), n, mode, ctypes.byref(r)))
            rs.append([n, 500 + i, 600 + i, mode, r.value])
    out["rse_cases"] = np.array(rs, np.float64)

    # --- multi_strategy_attention with a HeadCache (dispatch.cpp:30-91):
    # H=4, 256+44 tokens, d=64, B=64, plan [F, A0, A2, C] at t=1 after an all-Full t=0.
    H, nv, nt, d, B = 4, 256, 44, 64, 64
    n = nv + nt
    qs = [oracle.round_bf16(oracle.gaussian((H, n, d), 7000 + t * 10 + j)) for t in range(2) for j in range(3)]
    cache = ref().ref_cache_create()
    kinds0 = np.zeros(H, np.int32)
    wins0 = np.zeros(H, np.int64)
    o0 = np.zeros((H, n, d), np.float32)
    ref_check(ref().ref_multi_strategy_attention(ptr(qs[0], c_float), ptr(qs[1], c_float), ptr(qs[2], c_float), H,
                                                 d, nv, nt, 0, ptr(kinds0, c_int32), ptr(wins0, c_int64), cache, 0,
                                                 0, B, ptr(o0, c_float)))
    kinds1 = np.array([0, 1, 1, 2], np.int32)
    wins1 = np.array([0, 0, 2, 0], np.int64)
    o1 = np.zeros((H, n, d), np.float32)
    ref_check(ref().ref_multi_strategy_attention(ptr(qs[3], c_float), ptr(qs[4], c_float), ptr(qs[5], c_float), H,
                                                 d, nv, nt, 0, ptr(kinds1, c_int32), ptr(wins1, c_int64), cache, 0,
                                                 1, B, ptr(o1, c_float)))
    pa = []
    for h in range(H):
        t = c_int64()
        ref_check(ref().ref_cache_produced_at(cache, 0, h, ctypes.byref(t)))
        pa.append(t.value)
    ref().ref_cache_destroy(cache)
    out["msa_geom"] = np.array([H, nv, nt, d, B], np.int64)
    out["msa_out_t0"] = o0
    out["msa_out_t1"] = o1
    out["msa_produced_at"] = np.array(pa, np.int64)

    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), sum(v.nbytes for v in out.values()), "bytes")


if __name__ == "__main__":
    main()
