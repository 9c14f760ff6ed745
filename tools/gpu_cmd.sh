for r in 1 2 3 4; do timeout 300 python tools/e2e_probe.py --steps 40; DFA2_HOST_GROUPS_DESC=1 timeout 300 python tools/e2e_probe.py --steps 40 | sed 's/^/desc /'; done
