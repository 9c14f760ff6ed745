timeout 1200 python tools/ab_interleaved.py build/ab_cur10.so build/ab_merge.so --rounds 14 --plans FLUX68,flux_F,flux_A8,flux_C 2>&1 | tee gpurun_out/ab_merge.txt
DFA2_LIB=build/ab_merge.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
