timeout 600 python tools/sched_ab.py
