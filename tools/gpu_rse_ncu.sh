mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,launch__registers_per_thread,launch__occupancy_limit_registers --clock-control none -k regex:rse -c 40 --csv --log-file gpurun_out/rse_metrics.csv python tools/hbm_paths.py --ncu --out /tmp/x.json > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.DictReader(open('gpurun_out/rse_metrics.csv').read().split('\n',0)[0].splitlines()[[i for i,l in enumerate(open('gpurun_out/rse_metrics.csv').read().splitlines()) if l.startswith('"ID"')][0]:]))
for r in rows:
    print(r['ID'], r['Kernel Name'][:45], r['Metric Name'], r['Metric Value'])
PY
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('layer', d['layer_ms'], 'e2e', d['e2e'])"
