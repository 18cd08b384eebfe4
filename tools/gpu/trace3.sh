#!/bin/bash
# per-CTA tile stamps of the dX / dW GEMM launches (bf16)
PBRL_TC_TRACE=1 timeout 120 python tools/tc_trace.py --precision bf16 --dump 3 4 5 --out gpurun_out/trace_bf16_bwd.md > /dev/null 2>&1
