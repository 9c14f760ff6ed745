DFA2_RANDOM_LAYERS=400 timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k random 2>&1 | tail -3 | tee gpurun_out/random400.txt
