# usage: bash scripts/gpu_r02_gap.sh N TAG   (under gpurun --gpus N): one-clock breakdown + bench at NiN
N=${1:-2}; TAG=${2:-a}
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531"
timeout 300 $TR scripts/gap_coll.py --size 7600000 > gpurun_out/gap_${TAG}_n$N.jsonl 2> gpurun_out/gap_${TAG}_n$N.err
timeout 300 $TR scripts/gap_coll.py --size 65536 >> gpurun_out/gap_${TAG}_n$N.jsonl 2>> gpurun_out/gap_${TAG}_n$N.err
timeout 600 $TR bench.py --gpus $N --steps 100 --warmup 10 > gpurun_out/bench_${TAG}_n$N.json 2> gpurun_out/bench_${TAG}_n$N.err
timeout 900 python -m pytest tests/test_multi_gpu.py -x -q -m gpu -k "real_world_parity and not other" > gpurun_out/pytest_${TAG}_n$N.log 2>&1
echo "pytest exit=$?" >> gpurun_out/pytest_${TAG}_n$N.log
echo done
