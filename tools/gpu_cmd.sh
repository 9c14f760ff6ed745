timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_power.json 2> gpurun_out/bench_power.err; tail -2 gpurun_out/bench_power.err
python -c "import json;d=json.loads(open('gpurun_out/bench_power.json').read().strip().splitlines()[-1]);print(d['clocks'], d['layer_ms'], d['dense_ms'])"
nvidia-smi --query-gpu=power.limit,power.max_limit,power.default_limit,enforced.power.limit --format=csv
