#!/bin/bash
# usage: scripts/profile_kernel.sh <config> <kernel-regex> <tag> [p q]
# Runs ncu --set full on one count (2nd call) and writes, under gpurun_out/:
#   <tag>.ncu-rep, <tag>_sass.csv, <tag>_hot.txt (source-line hotspots), <tag>_summary.txt
set -u
cfg=$1; kre=$2; tag=$3; pq="${4:-} ${5:-}"
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$kre" -s 1 -c 1 \
    -o gpurun_out/$tag -f python scripts/one_count.py $cfg 2 $pq > gpurun_out/${tag}_run.log 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
mkdir -p /tmp/cub && (cd /tmp/cub && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2403_07858_b200/libbicount_b200.so >/dev/null 2>&1)
nvdisasm -g /tmp/cub/search.sm_100a.cubin > /tmp/cub/search.sass 2>/dev/null
kname=$(ncu -i gpurun_out/$tag.ncu-rep --page raw --csv 2>/dev/null | python -c "import csv,sys; r=list(csv.reader(sys.stdin)); print(r[2][r[0].index('Kernel Name')])")
mangled=$(grep -o '^\.text\.[^:]*' /tmp/cub/search.sass | sed 's/^\.text\.//' | python -c "
import sys,re
k=sys.argv[1]
base=re.search(r'::(\w+)<',k); base=base.group(1) if base else k.split('(')[0].split('::')[-1]
tpl=re.search(r'<([^>]*)>',k); args=[a.strip() for a in tpl.group(1).split(',')] if tpl else []
code=''.join('ELb1' if a in ('1','true','(bool)1') else 'ELb0' for a in args)
for l in sys.stdin:
    l=l.strip()
    if base in l and (not args or ('I'+code[1:]) in l or code in l): print(l); break
" "$kname")
python scripts/sass_hotspots.py gpurun_out/${tag}_sass.csv /tmp/cub/search.sass "$mangled" 40 > gpurun_out/${tag}_hot.txt 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page details --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keep=('Duration','Executed Ipc Active','Avg. Active Threads Per Warp','Registers Per Thread','Achieved Active Warps Per SM','L1/TEX Hit Rate','L2 Hit Rate','DRAM Throughput','Issue Slots Busy','Dynamic Shared Memory Per Block')
for row in r[1:]:
    d=dict(zip(h,row))
    if d['Metric Name'] in keep: print(d['Kernel Name'][:50], '|', d['Metric Name'], '=', d['Metric Value'], d['Metric Unit'])
" > gpurun_out/${tag}_summary.txt
cp paper_2403_07858_b200/csrc/search.cu gpurun_out/${tag}_search.cu
echo "kernel: $kname -> $mangled"
