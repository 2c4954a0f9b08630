#!/bin/bash
# ncu launch list (duration + DRAM/L2 bytes per launch) of one count, and a --set full
# capture of one kernel.  usage: scripts/ncu_launches.sh <tag> <kernel-regex> <cmd...>
set -u
tag=$1; kre=$2; shift 2
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
  --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv "$@" > gpurun_out/${tag}_launches_run.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:$kre" -c 1 \
  -o gpurun_out/${tag}_full -f "$@" > gpurun_out/${tag}_full_run.log 2>&1
echo "full capture rc=$?"
