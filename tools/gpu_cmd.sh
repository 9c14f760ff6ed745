for r in 1 2 3; do for g in 6 8 4 3; do DFA2_HOST_GROUPS=$g timeout 300 python tools/e2e_probe.py --steps 40 | sed "s/^/groups $g /"; done; done
