#!/bin/bash
# One measurement pass of the current build on a B200 (run under gpurun); everything
# lands in gpurun_out/meas/ and is summarised into profiles/r2/ afterwards:
#   launches_<cfg>.csv  ncu launch list of one count (duration, DRAM and L2 bytes per
#                       launch; --clock-control none; cold-cache, serialised)
#   full_<tag>.ncu-rep  ncu --set full of the dominant kernel (C5 triage enum_kernel,
#                       C5 sub_kernel, C2 LAZY enum_kernel)
#   b_<cfg>.json        bench.py lines (never taken under a profiler)
#   ref_C5.json         bench.py --impl reference (the CPU oracle port, sampled)
set -u
o=gpurun_out/meas
mkdir -p $o
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv"
for c in C5 C2 C4 C1; do
  timeout 900 ncu $M --log-file $o/launches_$c.csv python scripts/one_count.py $c 1 > $o/launches_$c.log 2>&1
  echo "launches $c rc=$?"
done
timeout 900 ncu $M --log-file $o/launches_C3_63.csv python scripts/one_count.py C3 1 6 3 > /dev/null 2>&1
timeout 900 ncu $M --log-file $o/launches_C3_36.csv python scripts/one_count.py C3 1 3 6 > /dev/null 2>&1
F="--set full --import-source on --clock-control none"
timeout 900 ncu $F -k regex:enum_kernel -s 0 -c 1 -o $o/full_c5_triage -f python scripts/one_count.py C5 1 > /dev/null 2>&1
timeout 900 ncu $F -k regex:sub_kernel -c 1 -o $o/full_c5_sub -f python scripts/one_count.py C5 1 > /dev/null 2>&1
timeout 900 ncu $F -k regex:rfilter_kernel -c 1 -o $o/full_c5_rfilter -f python scripts/one_count.py C5 1 > /dev/null 2>&1
timeout 900 ncu $F -k regex:l1_scatter -s 1 -c 1 -o $o/full_c5_l1fill -f python scripts/one_count.py C5 1 > /dev/null 2>&1
timeout 900 ncu $F -k regex:enum_kernel -s 1 -c 1 -o $o/full_c2_enum -f python scripts/one_count.py C2 2 > /dev/null 2>&1
echo "full captures done"
for c in C5 C2 C4 C1; do
  timeout 900 python bench.py --config $c > $o/b_$c.json 2> $o/b_$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --config C3 --p 6 --q 3 > $o/b_C3p6q3.json 2> $o/b_C3p6q3.err
timeout 900 python bench.py --config C3 --p 3 --q 6 > $o/b_C3p3q6.json 2> $o/b_C3p3q6.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $o/ref_C5.json 2> $o/ref_C5.err; echo "ref rc=$?"
