#!/bin/bash
# ncu evidence for the bench (run on the GPU box via gpurun), config $1 (default C3), round tag $2 (r02).
#  1) launch list of the bench command (cold, serialised: compare SHARES)
#  2) one --set full capture of the persistent executor kernel (the fused step, no phase launches),
#     exported as raw CSV and summarised with the library source sha (bench.py src_sha) so
#     bench.py only reports `traffic` from a capture of the build it times.
CFG=${1:-C3}
TAG=${2:-r02}
OUT=gpurun_out/ncu_$CFG
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu --no-phases > $OUT/launch_stdout.txt 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:serinv_exec -s 1 -c 1 \
  -o $OUT/prof python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu --no-phases > $OUT/full_stdout.txt 2>&1
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>&1
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>&1
ncu -i $OUT/prof.ncu-rep --page source --csv > $OUT/source.csv 2>&1
python tools/ncu_summary.py $OUT/raw.csv $CFG "bash tools/ncu_run.sh $CFG $TAG" > $OUT/summary.json
sz=$(stat -c %s $OUT/prof.ncu-rep 2>/dev/null || echo 0)
if [ "$sz" -gt 40000000 ]; then rm -f $OUT/prof.ncu-rep; fi
ls -la $OUT
