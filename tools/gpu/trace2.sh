#!/bin/bash
# phase timelines of the tcgen05 launches, bf16 mode, with and without C stores (diagnostics)
PBRL_TC_TRACE=1 timeout 120 python tools/tc_trace.py --precision bf16 --out gpurun_out/trace_bf16.md > /dev/null 2>&1
PBRL_TC_DBG=1 PBRL_TC_TRACE=1 timeout 120 python tools/tc_trace.py --precision bf16 --out gpurun_out/trace_bf16_nostore.md > /dev/null 2>&1
ls gpurun_out
