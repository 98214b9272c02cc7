#!/bin/bash
# launch list + ncu --set full summaries for profiles/ (run on the GPU box:
#   gpurun -- 'bash tools/full_profile.sh'; then python tools/summarize_profiles.py <tag>)
set -x
# launch list of the bench command itself (128K, 32 layers; one warm-up + one timed step)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv \
  --log-file gpurun_out/launches_full.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-approx \
  --no-decode > gpurun_out/launches_bench.log 2>&1
# one 128K prefill layer: stage 1 + stage 2 (rows >= 2048: attend_share_kernel)
ncu --set full --import-source on --clock-control none -k regex:"attend_share|select_tc" -s 2 -c 2 \
  -o gpurun_out/prefill128k -f python tools/profile_one.py 131072 > /dev/null 2>&1
# one batched-decode layer step (8 x 128K)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_cluster -s 5 -c 1 \
  -o gpurun_out/decode_cluster -f python tools/decode_probe.py 8 131072 1 > /dev/null 2>&1
# K1: the 128K prefill append + compress (first launch) and a re-sync pass
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stream_compress -c 2 \
  -o gpurun_out/compress -f python tools/compress_time.py 131072 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
