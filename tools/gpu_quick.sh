# gpu tests + bench line + hbm paths (no ncu). tag = $1
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 300 python tools/hbm_paths.py --out gpurun_out/hbm_$TAG.json 2>&1 | tail -8
