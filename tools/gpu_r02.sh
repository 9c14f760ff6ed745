# round-2 check: gpu tests (optionally a -k filter) + bench line. tag = $1, filter = $2
TAG=${1:-run}
FILTER=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -n "$FILTER" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$FILTER" 2>&1 | tail -25
else
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -25
fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -5 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
