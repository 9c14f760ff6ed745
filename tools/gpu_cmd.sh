timeout 900 python tools/configs_bench.py --only 1,2,3 --out gpurun_out/configs_r02i.json 2>&1 | grep -E "^cfg" | cut -c1-300
