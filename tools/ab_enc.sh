set -e
B=paper_2109_05410_b200
python -m pytest tests/test_gpu_codec.py tests/test_gpu_fp64.py -x -q > gpurun_out/codec_tests2.txt 2>&1 || true
for r in 1 2; do for v in minb4 minb5 minb6; do OOCZ_LIB=$PWD/$B/liboocz_ab_$v.so python tools/ab_one.py; done; done > gpurun_out/ab_enc.txt 2>&1
ncu --metrics smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active -k regex:zfp_ -c 4 python tools/prof_kernels.py > gpurun_out/ncu_enc2.txt 2>&1
