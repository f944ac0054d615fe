#!/bin/bash
# Instrumented libpsa (clock64 stamps in psa_attn_pp2_kernel, -DPSA_TRACE) for pp2_trace2.py.
set -e
cd "$(dirname "$0")/../.."
mkdir -p /tmp/psa_trace_build
for f in psa_abi psa_pyramid psa_importance psa_assign psa_attention psa_xlogits psa_permute psa_backward; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -Iinclude -DPSA_TRACE ${EXTRA} -c paper_2512_04025_b200/csrc/$f.cu -o /tmp/psa_trace_build/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/probes/libpsa_trace${TAG}.so /tmp/psa_trace_build/*.o
echo built scripts/probes/libpsa_trace${TAG}.so
