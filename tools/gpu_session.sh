#!/bin/bash
# One parameterised GPU session (run under gpurun): host info, the -m gpu suite
# (optionally a -k filter), smoke, and bench lines for the given configs.
#   bash tools/gpu_session.sh OUT "[pytest -k expr|all|none]" "C3 C2 ..." [extra bench args]
OUT=gpurun_out/${1:-session}
K=${2:-all}
CFGS=${3:-C3}
shift 3 2>/dev/null
EXTRA="$*"
mkdir -p $OUT
{ nproc; free -g; nvidia-smi --query-gpu=name,clocks.max.sm,power.limit,temperature.gpu --format=csv; } > $OUT/host.txt 2>&1
if [ "$K" != "none" ]; then
  if [ "$K" = "all" ]; then
    timeout 1800 python -m pytest tests -m gpu -q -rs > $OUT/gpu_tests.txt 2>&1; echo tests=$?
  else
    timeout 1800 python -m pytest tests -m gpu -q -rs -k "$K" > $OUT/gpu_tests.txt 2>&1; echo tests=$?
  fi
  tail -5 $OUT/gpu_tests.txt
  python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
fi
for c in $CFGS; do
  timeout 1200 python bench.py --config $c $EXTRA > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo bench_$c=$?
  tail -c 3000 $OUT/bench_$c.json
done
# optional traces: TRACE="selinv:365:2048:4 pobtaf:365:2048:4"
for t in $TRACE; do
  IFS=: read kind n b a P <<< "$t"
  timeout 600 python tools/trace.py $kind $n $b $a --P ${P:-1} > $OUT/trace_${kind}_${n}_${b}.txt 2>&1; echo trace_$t=$?
done
