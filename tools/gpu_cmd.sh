for rep in 1 2; do
for l in paper_2503_22796_b200/libdfa2_b200.so build/ab_mv_c16.so build/ab_mv_c8.so build/ab_mv_c4.so; do
  cp $l /tmp/libdfa2_b200.so
  echo "== $l $(LD_PRELOAD=/tmp/libdfa2_b200.so DFA2_HOST_PROFILE=1 timeout 300 tools/cpp_api_bench_bin 2>&1 | tail -2 | tr '\n' ' ')"
done
done
