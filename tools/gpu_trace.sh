python -m paper_2503_22796_b200.build --out /tmp/libtrace1.so -DDFA2_TRACE=1 > /dev/null 2>&1
python -m paper_2503_22796_b200.build --out /tmp/libtrace2.so -DDFA2_TRACE=2 > /dev/null 2>&1
for p in F A8; do echo "== FLUX $p trace1"; DFA2_LIB=/tmp/libtrace1.so timeout 120 python tools/trace_tiles.py $p; done
echo "== FLUX F trace2"; DFA2_TRACE_MODE=2 DFA2_LIB=/tmp/libtrace2.so timeout 120 python tools/trace_tiles.py F
echo "== SD3 F trace1"; DFA2_LIB=/tmp/libtrace1.so timeout 120 python tools/trace_tiles.py F --sd3
echo "== SD3 F trace2"; DFA2_TRACE_MODE=2 DFA2_LIB=/tmp/libtrace2.so timeout 120 python tools/trace_tiles.py F --sd3
