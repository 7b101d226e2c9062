RS_HOST_LANES=1 python tools/e2e_sweep.py 32:4 8:1 64:8 | sed 's/^/lanes1 /'
RS_HOST_LANES=2 python tools/e2e_sweep.py 32:4 8:1 64:8 16:2 | sed 's/^/lanes2 /'
