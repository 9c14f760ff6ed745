timeout 1200 python tools/ab_interleaved.py build/ab_cur4.so build/ab_rs184.so build/ab_rs200.so --rounds 14 --plans sd3_F,sd3_A16,sd3_A8,sd3_A2,sd3_A0 2>&1 | tee gpurun_out/ab_regsplit64.txt
