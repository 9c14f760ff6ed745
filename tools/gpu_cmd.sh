timeout 900 python tools/configs_bench.py --only 4 --out gpurun_out/cfg4_nosplit.json 2>&1 | grep cfg4 | cut -c1-400
DFA2_SPLIT_KV=1 timeout 900 python tools/configs_bench.py --only 4 --out gpurun_out/cfg4_split.json 2>&1 | grep cfg4 | cut -c1-400
