timeout 1200 python tools/ab_interleaved.py build/ab_cur2.so build/ab_sum2.so build/ab_sum4.so --rounds 14 --plans FLUX68,flux_F,sd3_F,sd3_A8,sd3_A0 2>&1 | tee gpurun_out/ab_sumchains.txt
