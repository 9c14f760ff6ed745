"""Generates tests/golden/plans/ from the REFERENCE ITSELF (plan JSON v1).

    make -C oracle all ref && python tests/golden/gen_plan_golden.py

For each seeded plan spec, the reference's own plan_to_json
(/root/reference/proj/src/plan.cpp:109-143, via oracle/ref_capi.cpp) writes
plan_<i>.json; cases.json records the spec. bad_cases.json records
malformed / invalid variants with the status the reference's plan_from_json
returns (6 = PlanValidationError, 1 = ShapeError, 0 = accepted).
"""
import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402
from oracle import c_int32, c_int64, ptr, ref  # noqa: E402

OUT = os.path.join(HERE, "plans")


def ref_json(spec):
    k = np.array(spec["kinds"], np.int32)
    w = np.array(spec["windows"], np.int64)
    ws = np.array(spec["window_set"] or [0], np.int64)
    n = c_int64()
    args = (spec["H"], spec["d"], spec["nv"], spec["nt"], spec["T"], spec["L"], spec["B"], spec["delta"],
            spec["coeff"], ptr(ws, c_int64), len(spec["window_set"]), ptr(k, c_int32), ptr(w, c_int64),
            spec["digest"].encode())
    oracle.ref_check(ref().ref_plan_to_json(*args, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    oracle.ref_check(ref().ref_plan_to_json(*args, buf, n.value + 1, ctypes.byref(n)))
    return buf.value.decode()


def ref_status(text):
    n = c_int64()
    k = np.zeros(1 << 16, np.int32)
    w = np.zeros(1 << 16, np.int64)
    return int(ref().ref_plan_from_json(text.encode(), len(k), ptr(k, c_int32), ptr(w, c_int64), ctypes.byref(n)))


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(2503)
    specs = []
    shapes = [(3, 8, 48, 8, 2, 2, 8), (24, 128, 16384, 512, 3, 4, 128), (24, 64, 4096, 333, 2, 3, 128),
              (4, 64, 1024, 77, 2, 1, 64), (1, 16, 17, 0, 1, 1, 4)]
    deltas = [0.4, 1.0, 0.0, 0.123456789, 1e-05]
    coeffs = [1.5, 1.0, 2.25, 100.0, 3.0]
    for i, (H, d, nv, nt, T, L, B) in enumerate(shapes):
        kinds, wins = [], []
        for t in range(T):
            for _ in range(L * H):
                k = int(rng.integers(0, 3 if t > 0 else 2))
                kinds.append(k)
                wins.append(int(rng.integers(0, 40)) if k == 1 else 0)
        digest = "" if i == 4 else ("%016x" % int(rng.integers(0, 2**62)))
        spec = {"H": H, "d": d, "nv": nv, "nt": nt, "T": T, "L": L, "B": B, "delta": deltas[i], "coeff": coeffs[i],
                "window_set": sorted({int(x) for x in rng.integers(0, 33, size=i + 1)}) if i != 4 else [],
                "kinds": kinds, "windows": wins, "digest": digest}
        text = ref_json(spec)
        with open(os.path.join(OUT, f"plan_{i}.json"), "w") as f:
            f.write(text)
        specs.append(spec)
    with open(os.path.join(OUT, "cases.json"), "w") as f:
        json.dump(specs, f)
    # malformed / invalid variants of plan_0 and the reference's verdict
    good = open(os.path.join(OUT, "plan_0.json")).read()
    bad = {
        "not_json": "{not json",
        "unknown_kind": good.replace('"full"', '"half"', 1),
        "bad_version": good.replace('"version": 1', '"version": 7', 1),
        "duplicate_entry": good.replace('"t": 1', '"t": 0', 1),
        "cached_at_t0": good.replace('"kind": "full"', '"kind": "cached"', 1),
        "missing_dims": good.replace('"dims"', '"dimz"', 1),
        "negative_window": good.replace('"window_blocks": ', '"window_blocks": -', 1),
        "zero_block": good.replace('"block": 8', '"block": 0', 1),
        "bad_delta": good.replace('"delta": 0.4', '"delta": -0.4', 1),
        "bad_coeff": good.replace('"coeff": 1.5', '"coeff": 0.5', 1),
        "zero_heads": good.replace('"H": 3', '"H": 0', 1),
        "short_heads": good.replace('{\n          "kind": "full"\n        },', '', 1),
        "trailing_garbage": good + "x",
        "float_ints": good.replace('"T": 2', '"T": 2.0', 1),
        "reordered_whitespace": json.dumps(json.loads(good)),
    }
    verdicts = {name: {"text": text, "status": ref_status(text)} for name, text in bad.items()}
    with open(os.path.join(OUT, "bad_cases.json"), "w") as f:
        json.dump(verdicts, f, indent=1)
    print({k: v["status"] for k, v in verdicts.items()})


if __name__ == "__main__":
    main()
