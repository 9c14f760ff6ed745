# A/B: build variants with -D flags on the box and bench each (FLUX68 + dense).
# usage: bash tools/gpu_ab.sh "NAME1:-DX=1 -DY=2" "NAME2:..." ...
mkdir -p gpurun_out/ab
timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  lib=/tmp/libdfa2_$name.so
  python -m paper_2503_22796_b200.build --out $lib $flags > /dev/null 2>&1 || { echo "$name: build failed"; continue; }
  DFA2_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/ab/$name.json 2>gpurun_out/ab/$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab/{n}.json"))
    print(f"{n:12s} layer {d['layer_ms']:.4f} ms  dense {d['dense_ms']:.4f} ms  computed {d['computed_tflops']:.0f} TF  frac {d['roofline']['frac']:.3f}  clk {d['clocks']['sm_mhz']}  e2e {d['e2e']['ms_per_step']:.3f}")
except Exception as e:
    print(n, "failed", e, open(f"gpurun_out/ab/{n}.err").read()[-500:])
PY
done
