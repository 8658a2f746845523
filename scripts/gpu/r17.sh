NCSG_SETUP_TIMES=1 python scripts/e2e_probe.py c3 2>&1 | tail -40
