timeout 1200 python tools/ab_interleaved.py build/ab_cur8.so build/ab_solo.so --rounds 14 --plans sd3_F,sd3_A16,sd3_A8,sd3_A2,sd3_A0 2>&1 | tee gpurun_out/ab_solo.txt
DFA2_LIB=build/lt5solo.so timeout 120 python tools/trace_skew.py F --sd3
DFA2_LIB=build/ab_solo.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
