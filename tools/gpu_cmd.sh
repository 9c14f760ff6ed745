for r in 1 2 3 4 5; do DFA2_HOST_STREAMS=1 timeout 300 python tools/e2e_probe.py --steps 40; timeout 300 python tools/e2e_probe.py --steps 40; done
