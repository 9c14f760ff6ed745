# HBM paths (RSE kernel, cached copy-back) + ncu captures of each
mkdir -p gpurun_out
TAG=${1:-run}
timeout 300 python tools/hbm_paths.py --out gpurun_out/hbm_$TAG.json 2>&1 | tail -8
timeout 600 ncu --set full --clock-control none -k regex:rse_partial -s 2 -c 1 -o gpurun_out/prof_rse_$TAG -f \
    python tools/hbm_paths.py --ncu --out /tmp/x.json > gpurun_out/ncu_rse_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/prof_copy_$TAG -f \
    python tools/hbm_paths.py --ncu --out /tmp/x.json > gpurun_out/ncu_copy_$TAG.log 2>&1
tail -2 gpurun_out/ncu_rse_$TAG.log gpurun_out/ncu_copy_$TAG.log
