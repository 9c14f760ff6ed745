# d=64 variants: smoke, parity, A/B (WIDE softmax on top of separate P + per-lane MMA warps)
mkdir -p gpurun_out
timeout 60 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -4
bash tools/gpu_ab2.sh "wide64:-DDFA2_WIDE64=1" "split:-DDFA2_WIDE64=0"
