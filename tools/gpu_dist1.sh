# the N > 1 bench code path (NCCL group, DistContext with Q, all-gather, max-over-ranks timing) at world size 1
mkdir -p gpurun_out/dist1
for c in C2 C4 C5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --dist --config $c --steps 3 --warmup 3 > gpurun_out/dist1/bench_$c.json 2> gpurun_out/dist1/bench_$c.err; echo $c=$?
done
cat gpurun_out/dist1/*.json; for f in gpurun_out/dist1/*.err; do tail -n 3 $f; done
