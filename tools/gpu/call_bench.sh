for d in 0 1 2 3; do echo "dbg $d"; DIPPM_RO_DBG=$d timeout 300 python tools/call_bench.py readout 2>&1 | tail -1; done
