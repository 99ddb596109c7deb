#!/bin/bash
# Round-2 ncu captures (run under gpurun; the reports land in gpurun_out/):
#  1. the launch list of the bench's C3 headline (serialised, cold-cache
#     per-launch durations: the kernels' shares of the step);
#  2. --set full of the three hot kernels on one C3-wide slab (4096^2 x 96
#     planes of the C3 data, rate 16; the stencil updates 64 planes = one
#     block at P = 64), for DRAM traffic vs algorithmic bytes and pipe use.
cd "$(dirname "$0")/.."
# (under ncu the 155 GB THP-registered arena got the process killed; the
#  launch list uses cudaHostAlloc for it: OOCZ_NO_THP=1)
OOCZ_NO_THP=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/${TAG:-r02}_launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --quick --no-c2 --no-cpu-baseline > gpurun_out/${TAG:-r02}_launches_c3_bench.json 2> gpurun_out/${TAG:-r02}_launches_c3_bench.err
N=4096 PLANES=96 REPS=2 ncu --set full --clock-control none --import-source on -k regex:"zfp_|stencil25" -c 6 -o gpurun_out/${TAG:-r02}_c3_kernels -f \
    python tools/prof_kernels.py > gpurun_out/${TAG:-r02}_c3_kernels.log 2>&1
PLANES=160 REPS=2 ncu --set full --clock-control none --import-source on -k regex:"zfp_|stencil25" -c 6 -o gpurun_out/${TAG:-r02}_c2_kernels -f \
    python tools/prof_kernels.py > gpurun_out/${TAG:-r02}_c2_kernels.log 2>&1
