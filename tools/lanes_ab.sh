#!/bin/bash
# c3 throughput vs lane count and CUDA_DEVICE_MAX_CONNECTIONS (run under gpurun)
for C in 8 16 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$C bash tools/variant_bench.sh 2>&1 | sed "s/^base /C$C-L3  /"
  CUDA_DEVICE_MAX_CONNECTIONS=$C DDH_LANES=4 DDH_RICD_PASSES=2 bash tools/variant_bench.sh 2>&1 | sed "s/^base /C$C-L4p /"
done
CUDA_DEVICE_MAX_CONNECTIONS=32 DDH_LANES=2 bash tools/variant_bench.sh 2>&1 | sed "s/^base /C32-L2  /"
