# launch list of the fused calibration pass vs the per-candidate passes (+ one full capture)
mkdir -p gpurun_out
TAG=${1:-fused}
timeout 300 python tools/influence_once.py 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:attn_fwd --csv --log-file gpurun_out/launches_$TAG.csv python tools/influence_once.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/prof_$TAG -f python tools/influence_once.py > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
