# one bench line + launch list + one full ncu capture of the fused kernel
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --ncu --no-cpu > /dev/null 2>&1
tail -5 gpurun_out/launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 \
    -o gpurun_out/prof_flux -f python bench.py --steps 1 --warmup 3 --ncu --no-cpu > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
