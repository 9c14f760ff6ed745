for rep in 1 2; do
for l in build/ab_onelaunch2.so paper_2503_22796_b200/libdfa2_b200.so; do
  cp $l /tmp/libdfa2_b200.so
  echo "== $l $(LD_PRELOAD=/tmp/libdfa2_b200.so DFA2_HOST_PROFILE=1 timeout 300 tools/cpp_api_bench_bin 2>&1 | tail -2 | tr '\n' ' ')"
done
done
timeout 900 python -m pytest tests/test_cpp_api.py tests/test_reference_suites.py -q -x -p no:cacheprovider 2>&1 | tail -1
