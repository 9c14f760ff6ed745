# the round-end driver sequence: smoke, GPU tests, bench (default), reference arm, launch list + ncu capture
TAG=${1:-final}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 600 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2>/dev/null; tail -c 300 gpurun_out/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_fwd -c 12 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --ncu --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 \
    -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 3 --ncu --no-cpu > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
