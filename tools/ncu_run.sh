#!/bin/bash
# ncu evidence for the bench (run on the GPU box via gpurun), config $1 (default C3), round tag $2 (r02),
# extra bench args after that (e.g. --engine sb).  Output kept small (gpurun copies back <= 64 MiB):
#  1) launch list of our kernels in the bench command (cold, serialised: compare SHARES)
#  2) one --set full capture of the first timed step's kernels (the executor, or the small-block
#     engine's launches), raw CSV + details + gzipped source page, summarised with the library
#     source sha (bench.py src_sha) so bench.py only reports `traffic` from a capture of the build
#     it times.
CFG=${1:-C3}
TAG=${2:-r02}
shift 2 2>/dev/null
EXTRA="$*"
SUF=""
case "$EXTRA" in *"--engine sb"*) SUF="_sb";; esac
OUT=gpurun_out/ncu_$CFG$SUF
mkdir -p $OUT
KRE='regex:serinv_exec|sb_factor|sb_inverse|sb_pre'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv --log-file $OUT/launches.csv \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu --no-phases $EXTRA > $OUT/launch_stdout.txt 2>&1
if [ -z "$SUF" ]; then SKIP=3; CNT=1; else SKIP=$(( $(grep -c sb_ $OUT/launches.csv) * 3 / 5 )); CNT=$(( $(grep -c sb_ $OUT/launches.csv) / 5 )); fi
timeout 1800 ncu --set full --clock-control none --import-source on -k "$KRE" -s $SKIP -c $CNT \
  -o $OUT/prof python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu --no-phases $EXTRA > $OUT/full_stdout.txt 2>&1
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>&1
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>&1
ncu -i $OUT/prof.ncu-rep --page source --csv 2>&1 | gzip -c > $OUT/source.csv.gz
python tools/ncu_summary.py $OUT/raw.csv $CFG "bash tools/ncu_run.sh $CFG $TAG $EXTRA" > $OUT/summary.json
rm -f $OUT/prof.ncu-rep
gzip -f $OUT/launches.csv
ls -la $OUT
