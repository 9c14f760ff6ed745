timeout 1200 python tools/ab_interleaved.py build/ab_cur5.so build/ab_e16.so build/ab_e0.so build/ab_e6.so --rounds 14 --plans FLUX68,flux_F,flux_A8 2>&1 | tee gpurun_out/ab_emu128b.txt
