timeout 1200 python tools/ab_interleaved.py build/ab_cur9.so build/ab_smma128.so --rounds 10 --plans FLUX68,flux_F,flux_A8 2>&1 | tee gpurun_out/ab_smma128.txt
