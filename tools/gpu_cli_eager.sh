#!/bin/bash
# Is the small-config gap a one-time lazy-module-loading cost? Same CLI A/B
# with CUDA_MODULE_LOADING=EAGER (kernels loaded at context creation).
export CUDA_MODULE_LOADING=EAGER
bash tools/gpu_cli_ab.sh "$@" | head -12
