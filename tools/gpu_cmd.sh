timeout 1200 python tools/ab_interleaved.py build/ab_refine.so build/ab_hh100.so build/ab_hh200.so --rounds 14 --plans FLUX68,flux_A8,flux_A2,flux_A0,LATE 2>&1 | tee gpurun_out/ab_halves128.txt
