for sep in 1 0; do
python -m paper_2503_22796_b200.build --out /tmp/lt1_$sep.so -DDFA2_TRACE=1 -DDFA2_SEP_P64=$sep > /dev/null 2>&1
python -m paper_2503_22796_b200.build --out /tmp/lt2_$sep.so -DDFA2_TRACE=2 -DDFA2_SEP_P64=$sep > /dev/null 2>&1
echo "== SEP=$sep SD3 F trace1"; DFA2_LIB=/tmp/lt1_$sep.so timeout 120 python tools/trace_tiles.py F --sd3
echo "== SEP=$sep SD3 F trace2"; DFA2_TRACE_MODE=2 DFA2_LIB=/tmp/lt2_$sep.so timeout 120 python tools/trace_tiles.py F --sd3
done
