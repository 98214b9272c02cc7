#!/bin/bash
# Build the stand-alone micro-benchmarks (binaries are git-ignored):
#   mma_bench  tcgen05.mma issue cost vs N, dependent vs independent accumulators
#   tma_bench  TMA random-block gather bandwidth
#   cluster_occupancy  co-resident clusters per cluster size
#   mufu_bench MUFU.EX2 vs FFMA throughput;  epi_bench  stage-1 epilogue in isolation
#   pipe_bench stage-1 MMA -> epilogue pipeline (+ TMA traffic) in isolation
set -e
cd "$(dirname "$0")"
for t in mma_bench tma_bench cluster_occupancy mufu_bench epi_bench pipe_bench; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o $t $t.cu
done
