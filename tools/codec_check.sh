#!/bin/bash
# Codec iteration on the GPU: bit-exact tests, isolated kernel times on one C2
# slab, and ncu instruction / pipe counts of the codec kernels (rate 16).
cd "$(dirname "$0")/.."
tag=${1:-x}
python -m pytest tests/test_gpu_codec.py tests/test_gpu_fp64.py -x -q > gpurun_out/codec_tests_$tag.txt 2>&1
python tools/time_kernels.py > gpurun_out/tk_$tag.json 2>&1
F64=1 ncu --metrics smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:zfp_ -c 4 python tools/prof_kernels.py > gpurun_out/ncu_$tag.txt 2>&1
