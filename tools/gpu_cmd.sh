timeout 1200 python tools/ab_interleaved.py build/ab_cur3.so paper_2503_22796_b200/libdfa2_b200.so --rounds 14 --plans FLUX68,flux_F,sd3_F,sd3_A8,sd3_A2,sd3_A0 2>&1 | tee gpurun_out/ab_maskregs.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
