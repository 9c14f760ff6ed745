timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "wide or padded or cache_miss" 2>&1 | tail -5
