for d in 0 64 1; do DIPPM_GEMM_DEBUG=$d timeout 300 python tools/gemm_probe.py fwd 2>&1 | grep "K=1024" | head -2; done
