# d=64 separate-P layout + per-lane MMA warps: smoke, parity, A/B
mkdir -p gpurun_out
timeout 60 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -4
bash tools/gpu_ab2.sh "split:-DDFA2_SEP_P64=1 -DDFA2_SPLIT_MMA64=1" "base:-DDFA2_SEP_P64=0"
