#!/bin/bash
# ncu --set full captures of the MiniCPM4-0.5B-shape kernels (16 q / 2 KV heads, d 64):
#   gpurun -- 'bash tools/profile_05b.sh'
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"attend_share|select_tc" -s 2 -c 2 \
  -o gpurun_out/prefill128k_05b -f python tools/profile_one.py 131072 16 2 64 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_cluster -s 5 -c 1 \
  -o gpurun_out/decode_05b -f python tools/decode_05b.py --steps 3 > /dev/null 2>&1
ls -la gpurun_out/*05b*.ncu-rep
