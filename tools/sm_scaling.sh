#!/bin/bash
# Stage-1 / stage-2 kernel time vs CTA count (one 128K layer): is stage 2 bound per SM or by aggregate L2?
for n in 148 111 96 74 56; do
  for k in select_tc attend_tc; do
    v=$(INFLLM2_SELECT_CTAS=$n INFLLM2_ATTEND_CTAS=$n ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$k -s 1 -c 1 --csv python tools/profile_one.py 131072 2>/dev/null | grep '^"' | tail -1 | awk -F'","' '{print $NF}' | tr -d '"')
    echo "ctas=$n $k ns=$v"
  done
done
