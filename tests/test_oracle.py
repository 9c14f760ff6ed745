"""Pins the plain-C oracle (oracle/oracle.c) to the reference itself:
golden vectors generated from the reference (tests/golden/gen_golden.py) and,
when oracle/_ref is built, live calls into the unmodified reference."""
import ctypes
import os

import numpy as np
import pytest

import oracle
from oracle import c_double, c_float, c_int32, c_int64, c_uint8, ptr

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def test_arrow_masks_bit_exact_against_reference_golden():
    for i in range(int(G["n_mask_cases"][0])):
        nv, nt, order, B, w = (int(x) for x in G[f"mask{i}_geom"])
        want = np.unpackbits(G[f"mask{i}_bits"])[: int(G[f"mask{i}_nbits"][0])]
        got = oracle.arrow_mask(nv, nt, order, B, w)
        assert np.array_equal(got, want), (nv, nt, order, B, w)
        ap = oracle.orc().orc_active_positions(ptr(got, c_uint8), nv + nt, B)
        assert ap == int(G[f"mask{i}_stats"][0])
        assert 4 * 64 * ap == int(G[f"mask{i}_stats"][1])


def test_reference_known_answers():
    # tests/test_arrow.cpp:53-66: 512+128, B=128, w=0 -> 13 active blocks, sparsity 0.48
    m = oracle.arrow_mask(512, 128, 0, 128, 0).reshape(5, 5)
    assert m.sum() == 13 and m[4].all() and m[:, 4].all() and m[0, 2] == 0
    ap = oracle.orc().orc_active_positions(ptr(np.ascontiguousarray(m.ravel()), c_uint8), 640, 128)
    assert abs(1 - ap / 640 ** 2 - 0.48) < 1e-12
    # window clamp (test_arrow.cpp:68-74)
    for w in (3, 4, 100):
        assert oracle.arrow_mask(512, 128, 0, 128, w).sum() == 25
    # text-first mirrors the band (test_arrow.cpp:83-92)
    t = oracle.arrow_mask(512, 128, 1, 128, 0).reshape(5, 5)
    assert t[0].all() and t[:, 0].all() and t.sum() == 13 and t[1, 3] == 0
    # test_bench.cpp:21-32 pinned sparsities at 4096+512
    for w, s in ((0, 0.7654), (6, 0.5015), (13, 0.2639)):
        mm = oracle.arrow_mask(4096, 512, 0, 128, w)
        ap = oracle.orc().orc_active_positions(ptr(mm, c_uint8), 4608, 128)
        assert abs((1 - ap / 4608 ** 2) - s) < 5e-5


def test_plan_flops_against_reference_golden():
    for name in ("cfg1", "cfg1_b64", "flux68", "sd3_flux68"):
        H, d, nv, nt, order, B, f = (int(x) for x in G[f"plan_{name}"])
        k = np.ascontiguousarray(G[f"plan_{name}_kinds"])
        w = np.ascontiguousarray(G[f"plan_{name}_windows"])
        got = oracle.orc().orc_plan_flops(H, d, nv, nt, order, B, ptr(k, c_int32), ptr(w, c_int64))
        assert got == f, name
    # survey numbers: FLUX68 = 1,127.2 GFLOP, reduction 0.6787
    H, d, nv, nt, order, B, f = (int(x) for x in G["plan_flux68"])
    dense = 24 * 4 * 128 * 16896 ** 2
    assert abs(f / 1e9 - 1127.2) < 0.1 and abs(1 - f / dense - 0.6787) < 1e-4


def test_sparse_forward_and_f64_oracle_against_reference_golden():
    for i in range(int(G["n_att_cases"][0])):
        nv, nt, d, B, w, seed = (int(x) for x in G[f"att{i}_geom"])
        n = nv + nt
        q, k, v = (oracle.gaussian((n, d), seed + j) for j in range(3))
        m = oracle.arrow_mask(nv, nt, 0, B, w)
        want64 = G[f"att{i}_ref_f64"]
        got64 = oracle.attention_rows_f64(q, k, v, m, B)
        # same operation order as attention_head_impl<double> (tensor.cpp:73-114): bit-exact
        assert np.array_equal(got64, want64), i
        o32 = np.zeros((n, d), np.float32)
        rc = oracle.orc().orc_sparse_forward_f32(ptr(q, c_float), ptr(k, c_float), ptr(v, c_float),
                                                 ptr(o32, c_float), n, d, ptr(m, c_uint8), B)
        assert rc == 0
        ref32 = G[f"att{i}_sparse_f32"]
        scale = np.abs(want64).max()
        # reference desk threshold: <= 1e-5 relative to the f64 oracle
        assert np.abs(o32 - want64).max() / scale < 1e-5
        assert np.abs(ref32 - want64).max() / scale < 1e-5
        assert np.abs(o32 - ref32).max() / scale < 1e-5


def test_rse_bit_exact_against_reference_golden():
    for n, s1, s2, mode, want in G["rse_cases"]:
        a = oracle.gaussian((int(n),), int(s1))
        b = oracle.gaussian((int(n),), int(s2)) * 0.1 + a
        assert oracle.rse_f32(b, a, int(mode)) == want


def test_rse_hand_values():
    # tests/test_calibrate.cpp:48-72
    assert oracle.rse_f32(np.array([2, 2], np.float32), np.array([1, 3], np.float32)) == pytest.approx(1.0)
    y = np.array([1, 3], np.float32)
    assert oracle.rse_f32(y, y, 0) == 0.0
    assert oracle.rse_f32(y, y, 1) == pytest.approx(1.0)
    with pytest.raises(RuntimeError):
        oracle.rse_f32(np.array([5, 6], np.float32), np.array([5, 5], np.float32))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_on_random_geometries():
    rng = np.random.default_rng(99)
    L = oracle.ref()
    for _ in range(200):
        nv, nt = int(1 + rng.integers(400)), int(rng.integers(80))
        order, B, w = int(rng.integers(2)), int(1 + rng.integers(140)), int(rng.integers(8))
        nb = c_int64()
        oracle.ref_check(L.ref_arrow_mask(1, 8, nv, nt, order, B, w, None, ctypes.byref(nb)))
        want = np.zeros(nb.value ** 2, np.uint8)
        oracle.ref_check(L.ref_arrow_mask(1, 8, nv, nt, order, B, w, ptr(want, c_uint8), ctypes.byref(nb)))
        assert np.array_equal(oracle.arrow_mask(nv, nt, order, B, w), want)
