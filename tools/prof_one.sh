#!/bin/bash
# One ncu --set full capture of selected kernels of one bench workload, exported
# to CSV on the box (run under gpurun; the plain run must exit 0 first).
#   tools/prof_one.sh <tag> <workload> <kernel regex> <count>
set -u
TAG=$1; WL=$2; KR=$3; CNT=$4
mkdir -p gpurun_out
CMD="python bench.py --workload $WL --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --serial"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$TAG.log; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"$KR" -c $CNT \
    -o gpurun_out/$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>/dev/null
gzip -f gpurun_out/${TAG}_source.csv
rm -f gpurun_out/$TAG.ncu-rep
echo done
