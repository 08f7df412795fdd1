#!/bin/bash
# Update-kernel A/B: GPU parity subset for the update kernels, then short
# benches of the TMA-staged (default) and LDG update kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "update_kernels or parity_build or fma_build" > gpurun_out/pytest_upd.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_upd.log
NO_PYTEST=1 bash tools/gpu_ab.sh "$@" 2>&1 | grep -v "^pytest\|passed\|^\.\.\." 
