for a in 0 592 1184 296; do HUSKY_GATHER_AHEAD=$a timeout 300 python tools/c5_probe.py 30 2 C5 2>&1 | tail -1; done
HUSKY_GATHER_AHEAD=0 timeout 300 python tools/c5_probe.py 27 3 C5 2>&1 | tail -1
timeout 300 python tools/c5_probe.py 27 3 C5 2>&1 | tail -1
