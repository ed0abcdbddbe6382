# usage: bash scripts/gpu_bench.sh N tag   — driver-style bench runs (ours + reference arm)
N=${1:-1}; TAG=${2:-r}
if [ "$N" = "1" ]; then
  python bench.py --impl reference > gpurun_out/bench_${TAG}_ref_n1.json 2> gpurun_out/bench_${TAG}_ref_n1.err
  python bench.py > gpurun_out/bench_${TAG}_n1.json 2> gpurun_out/bench_${TAG}_n1.err
else
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29514"
  timeout 600 $TR bench.py --gpus $N > gpurun_out/bench_${TAG}_n$N.json 2> gpurun_out/bench_${TAG}_n$N.err
  for c in googlenet alexnet vgg19; do
    timeout 600 $TR bench.py --gpus $N --config $c --steps 50 --warmup 5 --no-baselines > gpurun_out/bench_${TAG}_n${N}_$c.json 2> gpurun_out/bench_${TAG}_n${N}_$c.err
  done
fi
