DFA2_LIB=build/ab_rseslow.so timeout 120 python tools/rse_bits.py > gpurun_out/rse_slow.txt 2>&1
timeout 120 python tools/rse_bits.py > gpurun_out/rse_fast.txt 2>&1
cmp gpurun_out/rse_slow.txt gpurun_out/rse_fast.txt && echo BITWISE_EQUAL; cat gpurun_out/rse_fast.txt | cut -c1-200
for r in 1 2; do for l in build/ab_rseslow.so paper_2503_22796_b200/libdfa2_b200.so; do echo "== $l"; DFA2_LIB=$l timeout 300 python tools/hbm_paths.py 2>&1 | grep "rse bf16"; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_calibration_gpu.py -m gpu -q -x -p no:cacheprovider -k "rse or influence" 2>&1 | tail -1
