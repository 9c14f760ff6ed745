"""SHA-256 of the REFERENCE's generate() streams (src/workload.cpp:120-228 via
oracle/ref_capi.cpp) for a few configs -> tests/golden/workload_golden.json.
Layout hashed: raw f32 q|k|v of every (t, layer) slot, t-major.

    make -C oracle all ref && python tests/golden/gen_workload_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402
from oracle import c_float, ptr, ref  # noqa: E402

CONFIGS = [  # H, d, nv, nt, order, L, T, B, seed (reference tests' desk/tiny/small configs + cfg1 geometry)
    (4, 8, 48, 8, 0, 2, 3, 8, 9),
    (8, 32, 256, 32, 0, 4, 8, 32, 1234),
    (3, 16, 100, 12, 1, 2, 2, 16, 77),
    (4, 64, 1024, 77, 0, 1, 2, 128, 1234),
]


def main():
    out = []
    for (H, d, nv, nt, order, L, T, B, seed) in CONFIGS:
        per = H * (nv + nt) * d
        q, k, v = (np.zeros(T * L * per, np.float32) for _ in range(3))
        oracle.ref_check(ref().ref_generate(H, d, nv, nt, order, L, T, B, seed, ptr(q, c_float), ptr(k, c_float),
                                            ptr(v, c_float)))
        h = hashlib.sha256()
        for s in range(T * L):
            for x in (q, k, v):
                h.update(x[s * per:(s + 1) * per].tobytes())
        out.append({"config": [H, d, nv, nt, order, L, T, B, seed], "sha256": h.hexdigest()})
    with open(os.path.join(HERE, "workload_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(out)


if __name__ == "__main__":
    main()
