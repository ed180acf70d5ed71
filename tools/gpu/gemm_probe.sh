for k in fwd pool; do DIPPM_GEMM_DEBUG=0 timeout 300 python tools/gemm_probe.py $k 2>&1 | grep "K=1024" | head -2; done
