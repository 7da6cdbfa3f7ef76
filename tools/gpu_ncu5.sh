# ncu --set full of the C5 (small-b) bench launch + bench lines carrying roofline_hbm
OUT=gpurun_out/ncu_C5
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:serinv_exec -s 1 -c 1 \
  -o $OUT/prof python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/full_stdout.txt 2>&1; echo ncu=$?
ncu -i $OUT/prof.ncu-rep --page raw --csv > $OUT/raw.csv 2>&1
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv 2>&1
rm -f $OUT/prof.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:serinv_exec --csv --log-file $OUT/launches.csv \
  python bench.py --config C5 --steps 2 --warmup 1 --no-e2e --no-cpu > $OUT/launch_stdout.txt 2>&1; echo launches=$?
mkdir -p gpurun_out/final3
for c in C5 C2; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/final3/bench_$c.json 2> gpurun_out/final3/bench_$c.err; echo $c=$?
done
cat gpurun_out/final3/*.json
ls -la $OUT
