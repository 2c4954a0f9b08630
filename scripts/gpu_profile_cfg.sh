#!/bin/bash
# ncu evidence for one config on the current build, all under gpurun_out/<tag>/:
#   launches.csv  -- every launch of one count (duration, DRAM/L2 bytes), --clock-control none
#   full.ncu-rep  -- --set full of the top kernels (regex), first count
# usage: scripts/gpu_profile_cfg.sh <tag> <config> <kernel-regex> [count-of-kernels]
set -u
tag=$1; cfg=$2; kre=$3; n=${4:-3}
out=gpurun_out/$tag
mkdir -p $out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
  --clock-control none --csv --log-file $out/launches.csv python scripts/one_count.py $cfg 1 > $out/launches_run.log 2>&1
echo "launch list rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k "regex:$kre" -c $n \
  -o $out/full -f python scripts/one_count.py $cfg 1 > $out/full_run.log 2>&1
echo "full capture rc=$?"
