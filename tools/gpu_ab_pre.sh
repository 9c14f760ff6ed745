# A/B over PREBUILT libraries build/ab_<name>.so (built here, shipped with the snapshot):
# FLUX68 + dense through bench.py, then the SD3 and FLUX plan-kind sweeps.
# usage: bash tools/gpu_ab_pre.sh name1 name2 ...
mkdir -p gpurun_out/ab
for name in "$@"; do
  lib=build/ab_$name.so
  DFA2_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/ab/$name.json 2>gpurun_out/ab/$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab/{n}.json"))
    print(f"{n:12s} layer {d['layer_ms']:.4f} ms  dense {d['dense_ms']:.4f} ms  computed {d['computed_tflops']:.0f} TF  frac {d['roofline']['frac']:.3f}  clk {d['clocks']['sm_mhz']}", flush=True)
except Exception as e:
    print(n, "failed", e, open(f"gpurun_out/ab/{n}.err").read()[-800:])
PY
  DFA2_LIB=$lib timeout 300 python tools/plan_sweep.py --sd3 --steps 20 2>&1 | grep -v commit=1 | sed "s/^/  sd3 /"
  DFA2_LIB=$lib timeout 300 python tools/plan_sweep.py --steps 10 2>&1 | grep -E "all_A0|all_A8|all_F |FLUX68 " | grep -v "commit=0" | sed "s/^/  flux /"
done
