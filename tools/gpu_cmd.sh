timeout 1200 python tools/ab_interleaved.py build/ab_cur6.so build/ab_ctlsleep.so --rounds 14 --plans FLUX68,flux_F,flux_A8,sd3_F,sd3_A8,sd3_A2,sd3_A0,flux_C 2>&1 | tee gpurun_out/ab_ctlsleep.txt
