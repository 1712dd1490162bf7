#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; each ncu only after the same command exited 0 plain).
# Raw .ncu-rep files are exported to CSV on the box and deleted (64 MiB return limit).
set -u
mkdir -p gpurun_out
export_rep() {  # $1 = report base name
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
  gzip -f gpurun_out/$1_source.csv
  rm -f gpurun_out/$1.ncu-rep
}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --streams 0"
$CMD > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --kernel-name-base function \
    --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch_c2.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base function \
    -k regex:"k_rc_small_encode|k_rc_small_decode|k_enc_uchan128|k_dec_uchan128|k_enc128|k_dec128|k_gather" -c 7 \
    -o gpurun_out/prof_c2_r1 $CMD > gpurun_out/ncu_full_c2.log 2>&1 && export_rep prof_c2_r1
CMD1="python bench.py --workload c1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --streams 0"
$CMD1 > gpurun_out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"k_enc128|k_dec128" -c 2 \
    -o gpurun_out/prof_c1_r1 $CMD1 > gpurun_out/ncu_full_c1.log 2>&1 && export_rep prof_c1_r1
CMD5="python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --streams 0"
$CMD5 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"k_rc_large" -c 2 \
    -o gpurun_out/prof_c5_r1 $CMD5 > gpurun_out/ncu_full_c5.log 2>&1 && export_rep prof_c5_r1
du -sh gpurun_out
echo done
