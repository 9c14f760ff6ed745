timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err; tail -2 gpurun_out/bench_r02f.err; python -c "
import json; d=json.load(open('gpurun_out/bench_r02f.json')); print(d['layer_ms'], d['roofline']['frac'], d['clocks'], d['parity']['pass'], d['e2e']['ms_per_step'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 4 -c 1 -o gpurun_out/flux68_r02f_full python bench.py --steps 2 --warmup 3 --ncu > /dev/null 2>&1; echo ncu $?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02f.csv python bench.py --steps 2 --warmup 3 --ncu > /dev/null 2>&1; echo ncu2 $?
