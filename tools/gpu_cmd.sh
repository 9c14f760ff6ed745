timeout 1200 python tools/ab_interleaved.py paper_2503_22796_b200/libdfa2_b200.so build/ab_p1.so build/ab_d1.so build/ab_pd.so --rounds 14 --plans FLUX68,flux_F,flux_A8,flux_A0,LATE 2>&1 | tee gpurun_out/ab_mma.txt
for l in ab_pd ab_d1; do DFA2_LIB=build/$l.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1; done
