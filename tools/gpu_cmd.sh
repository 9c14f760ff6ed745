timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r02j.json 2> gpurun_out/bench_r02j.err; tail -2 gpurun_out/bench_r02j.err
python -c "import json;d=json.loads(open('gpurun_out/bench_r02j.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['clocks'], d['parity']['pass'], d.get('e2e_cpp_f32',{}).get('ms_per_step'))"
