timeout 300 python tools/api_overhead.py 2>&1 | head -3
timeout 120 python tools/allc_probe.py flux; timeout 120 python tools/allc_probe.py sd3
timeout 300 python tools/hbm_paths.py 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
