#!/bin/bash
# full bench line + launch list + ncu summaries for profiles/
set -x
python bench.py > gpurun_out/bench_full.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_full.csv python bench.py --seq 32768 --layers 2 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"attend_tc|select_tc" -s 2 -c 2 -o gpurun_out/prefill128k python tools/profile_one.py 131072 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:decode_cluster -s 5 -c 1 -o gpurun_out/decode_cluster python tools/decode_probe.py 8 131072 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
