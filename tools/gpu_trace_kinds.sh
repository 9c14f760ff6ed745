# per-tile timelines (TRACE=1 build prebuilt at build/lt1.so) for plan kinds at FLUX d=128 and SD3 d=64
for p in F A16 A8 A2 A0; do echo "== FLUX $p"; DFA2_TRACE_PCT=1 DFA2_LIB=build/lt1.so timeout 120 python tools/trace_tiles.py $p; done
echo "== FLUX68"; DFA2_TRACE_PCT=1 DFA2_LIB=build/lt1.so timeout 120 python tools/trace_tiles.py "F A8 C A0 F A8 C A8 F A8 C A0 F A8 C A0 F A8 C A8 F A8 C A0"
for p in F A8 A0; do echo "== SD3 $p"; DFA2_TRACE_PCT=1 DFA2_LIB=build/lt1.so timeout 120 python tools/trace_tiles.py $p --sd3; done
