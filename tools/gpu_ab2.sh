# A/B: build variants with -D flags on the box; per variant: FLUX68 bench line
# (layer/dense ms) + SD3 (d=64) all-Full / Arrow sweep from configs_bench.
# usage: bash tools/gpu_ab2.sh "NAME1:-DX=1 -DY=2" "NAME2:..." ...
mkdir -p gpurun_out/ab
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  lib=/tmp/libdfa2_$name.so
  python -m paper_2503_22796_b200.build --out $lib $flags > /dev/null 2>&1 || { echo "$name: build failed"; continue; }
  DFA2_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/ab/$name.json 2>gpurun_out/ab/$name.err
  DFA2_LIB=$lib timeout 300 python tools/configs_bench.py --only 2 --out gpurun_out/ab/${name}_sd3.json > /dev/null 2>&1
  DFA2_LIB=$lib timeout 120 python tools/cached_layer_bench.py > gpurun_out/ab/${name}_cached.txt 2>&1
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab/{n}.json"))
    s = json.load(open(f"gpurun_out/ab/{n}_sd3.json"))["cfg2_sd3_window_sweep"]
    sd3 = " ".join(f"{r['plan'].replace('all ','')}={r['ms']*1e3:.0f}us/{r['computed_tflops']:.0f}TF" for r in s)
    cached = open(f"gpurun_out/ab/{n}_cached.txt").read().strip()
    print(f"{n:10s} FLUX68 {d['layer_ms']:.4f} ms dense {d['dense_ms']:.4f} ms ({d['computed_tflops']:.0f} TF, clk {d['clocks']['sm_mhz']}) | {cached} | SD3 {sd3}")
except Exception as e:
    print(n, "failed", e, open(f"gpurun_out/ab/{n}.err").read()[-800:])
PY
done
