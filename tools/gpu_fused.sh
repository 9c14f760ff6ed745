# fused calibration pass: parity tests, per-layer timing, configs 5, FLUX regression check
mkdir -p gpurun_out
TAG=${1:-fused}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -6
timeout 300 python tools/influence_once.py 2>&1 | tail -4
timeout 600 python tools/configs_bench.py --only 5 --out gpurun_out/configs5_$TAG.json 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('layer_ms', d['layer_ms'], 'dense', d['dense_ms'])"
