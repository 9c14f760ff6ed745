for l in lt5 lt5sw; do echo "== $l"; DFA2_LIB=build/$l.so timeout 120 python tools/trace_skew.py F --sd3; DFA2_LIB=build/$l.so timeout 120 python tools/trace_skew.py F; done
