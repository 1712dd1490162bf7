#!/bin/bash
# Round measurement set (run under gpurun from the repo root): bench lines for
# every workload, the reference arm, the c2 launch list and ncu --set full
# captures of the dominant kernels (each only after its plain run exited 0).
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
python bench.py --workload c1 --steps 20 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --workload c3 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --workload c5 --steps 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
# launch list of the default bench (cold-cache, serialised: shares only)
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --streams 0"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --kernel-name-base function \
    --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1
tools/prof_one.sh prof_c2 c2 "k_fused|k_gather" 6
tools/prof_one.sh prof_c1 c1 "k_enc128|k_dec128" 4
tools/prof_one.sh prof_c5 c5 "k_rc_large|k_enc128|k_dec128" 8
du -sh gpurun_out
echo done
