#!/bin/bash
PBRL_TC_TRACE=1 timeout 120 python tools/tc_trace.py --precision bf16 --out gpurun_out/trace_bf16.md > /dev/null 2>&1
