#!/bin/bash
# Development helper: TMA stage-count variants of libnlsp_gpu (NLSP_GPU_LIB=...).
set -e
D=$(cd "$(dirname "$0")/.." && pwd)/paper_2601_20174_b200
mkdir -p $D/variants $D/build/variants
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$D/../include -I$D/csrc"
make -s -C $D
for spec in "$@"; do
  tag=t_$(echo $spec | tr ',' '_')
  IFS=, read SS RS G U <<< "$spec"
  $NV -DNLSP_SPMV_STAGES=$SS -DNLSP_RESTRICT_STAGES=$RS -DNLSP_SPMV_G=${G:-1} -DNLSP_SPMV_U=${U:-1} -c $D/csrc/solve_kernels.cu -o $D/build/variants/solve_$tag.o &
done
wait
for spec in "$@"; do
  tag=t_$(echo $spec | tr ',' '_')
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/variants/libnlsp_gpu_$tag.so $D/build/variants/solve_$tag.o $D/build/setup_kernels.o $D/build/nlsp_gpu.o -lcudart
done
ls $D/variants
