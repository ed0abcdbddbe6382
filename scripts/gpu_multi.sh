# usage: bash scripts/gpu_multi.sh N   (run under gpurun --gpus N)
N=${1:-2}
set -x
nvidia-smi topo -m > gpurun_out/topo_n$N.txt 2>&1
timeout 900 python -m pytest tests/test_multi_gpu.py -x -q -m gpu > gpurun_out/pytest_mgpu_n$N.log 2>&1
echo "pytest exit=$?" >> gpurun_out/pytest_mgpu_n$N.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"
timeout 600 $TR bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
for c in googlenet alexnet vgg19; do
  timeout 600 $TR bench.py --gpus $N --config $c --steps 50 --warmup 5 > gpurun_out/bench_n${N}_$c.json 2> gpurun_out/bench_n${N}_$c.err
done
echo done
