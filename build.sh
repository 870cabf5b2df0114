#!/bin/bash
# Builds libppx.so (sm_100a) in-tree. Invoked by __graft_entry__.build().
set -e
cd "$(dirname "$0")"
NCCL=$(python -c "import nvidia.nccl,os;print(os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0])")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I"$NCCL/include" -L"$NCCL/lib" -l:libnccl.so.2 -Xlinker -rpath="$NCCL/lib" \
  $PPX_NVCC_EXTRA paper_2508_00960_b200/csrc/ppx.cu -o "${PPX_OUT:-paper_2508_00960_b200/libppx.so}"
