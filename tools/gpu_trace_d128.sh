python -m paper_2503_22796_b200.build --out /tmp/lt1.so -DDFA2_TRACE=1 > /dev/null 2>&1
for p in F A8 A0; do echo "== FLUX $p"; DFA2_TRACE_PCT=1 DFA2_LIB=/tmp/lt1.so timeout 120 python tools/trace_tiles.py $p; done
echo "== FLUX68"; DFA2_TRACE_PCT=1 DFA2_LIB=/tmp/lt1.so timeout 120 python tools/trace_tiles.py "F A8 C A0 F A8 C A8 F A8 C A0 F A8 C A0 F A8 C A8 F A8 C A0"
