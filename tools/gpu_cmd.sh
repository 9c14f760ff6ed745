P="F F F F F F A8 A8 A8 A8 A8 A8 A0 A0 A0 A0 A0 A0 C C C C C C"
for r in 1 2; do for l in build/ab_eqgroups.so paper_2503_22796_b200/libdfa2_b200.so; do
  DFA2_LIB=$l timeout 300 python tools/e2e_probe.py --steps 30 | sed "s|^|$(basename $l) |"
  DFA2_LIB=$l timeout 300 python tools/e2e_probe.py --steps 30 --plan "$P" | sed "s|^|$(basename $l) |"
done; done
