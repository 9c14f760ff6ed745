for n in r_base r_c4 r_s2k16 r_c4s3 r_c6s2; do echo "== $n"; DFA2_LIB=build/ab_$n.so timeout 300 python tools/hbm_paths.py --out gpurun_out/hbm_$n.json 2>&1 | grep rse; done
