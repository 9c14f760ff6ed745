for p in F; do echo "== FLUX $p"; DFA2_LIB=build/lt3.so timeout 120 python tools/trace_timeline.py $p 40 4; done
