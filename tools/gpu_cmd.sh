for r in 1 2; do
for l in build/ab_rse0.so paper_2503_22796_b200/libdfa2_b200.so; do echo "== $l"; DFA2_LIB=$l timeout 300 python tools/hbm_paths.py 2>&1 | grep rse; done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_calibration_gpu.py -m gpu -q -x -p no:cacheprovider -k "rse or influence" 2>&1 | tail -1
