timeout 1200 python tools/ab_interleaved.py build/ab_lpt.so build/ab_refine.so --rounds 14 --plans FLUX68,flux_F,flux_A8,flux_A0,sd3_F,sd3_A16,sd3_A8,sd3_A4,sd3_A2,sd3_A1,sd3_A0 2>&1 | tee gpurun_out/ab_refine.txt
for l in ab_lpt ab_refine; do echo "== $l"; DFA2_LIB=build/$l.so timeout 300 python tools/plan_miss_bench.py 2>&1 | tail -4; done | tee gpurun_out/plan_miss_refine.txt
DFA2_LIB=build/lt4.so timeout 300 python tools/cta_tail.py --sd3 F A16 A8 A4 A2 A0 2>&1 | tee gpurun_out/cta_refine_sd3.txt
DFA2_LIB=build/lt4.so timeout 300 python tools/cta_tail.py F A8 A0 FLUX68 2>&1 | tee gpurun_out/cta_refine_flux.txt
