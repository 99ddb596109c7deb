#!/bin/bash
# compute-sanitizer passes over the kernels (run under gpurun); summary lines
# to gpurun_out/sanitizer.md (profiles/r02_sanitizer.md)
cd "$(dirname "$0")/.."
S=/usr/local/cuda/bin/compute-sanitizer
run() { name=$1; shift; echo "## $name"; echo '```'; timeout 900 "$@" 2>&1 | grep -E "COMPUTE-SANITIZER|ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Invalid|Race|hazard|smoke" | head -20; echo "rc=${PIPESTATUS[0]}"; echo '```'; }
{
run memcheck_smoke $S --tool memcheck python -c "import __graft_entry__ as g; g.smoke()"
run memcheck_codec $S --tool memcheck python -m pytest tests/test_gpu_codec.py -q -k "encode_bit_exact or decode_bit_exact or arbitrary" -x
run initcheck_codec $S --tool initcheck python -m pytest tests/test_gpu_codec.py -q -k "encode_bit_exact and 16" -x
run racecheck_codec $S --tool racecheck python -m pytest tests/test_gpu_codec.py -q -k "random_shapes" -x
run synccheck_codec $S --tool synccheck python -m pytest tests/test_gpu_codec.py -q -k "random_shapes" -x
run memcheck_fp64 $S --tool memcheck python -m pytest tests/test_gpu_fp64.py -q -k "encode64 or decode64" -x
run initcheck_fp64 $S --tool initcheck python -m pytest tests/test_gpu_fp64.py -q -k "encode64_bit_exact" -x
run racecheck_stencil $S --tool racecheck python -m pytest tests/test_gpu_stencil.py -q -x
run memcheck_engine $S --tool memcheck python -m pytest tests/test_gpu_engine.py -q -k "stepper_matches_oracle" -x
run memcheck_hostmem $S --tool memcheck python -m pytest tests/test_gpu_hostmem.py -q -x
} > gpurun_out/sanitizer.md
