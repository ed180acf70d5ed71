for d in 4 132 0 128; do DIPPM_GEMM_DEBUG=$d timeout 300 python tools/gemm_probe.py fwd 2>&1 | grep "K=1024" | head -2; done
