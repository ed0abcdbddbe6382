# usage: bash scripts/gpu_r02_exit.sh N   (under gpurun --gpus N): exit protocol push vs poll (A/B/A/B),
# one-clock breakdown at NiN size, real-world parity first
N=${1:-2}
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for E in poll push; do
  FC_EXIT=$E FC_MP_TIMEOUT=5 FC_MP_TIMEOUT_TEST=0 FC_MP_STRESS=300 timeout 600 $TR --master-port 29541 tests/mp_worker.py > gpurun_out/r02_exit_mp_${E}_n$N.log 2>&1
  echo "$E parity rc=$? ok=$(grep -c MP_OK gpurun_out/r02_exit_mp_${E}_n$N.log)" >> gpurun_out/r02_exit_n$N.txt
done
grep NCCL_TOL gpurun_out/r02_exit_mp_poll_n$N.log >> gpurun_out/r02_exit_n$N.txt
for rep in 1 2; do for E in poll push; do
  FC_EXIT=$E timeout 300 $TR --master-port 29542 scripts/gap_coll.py --size 7600000 --dump 2>/dev/null | grep '"fused"' | sed "s/^/$E rep$rep /" >> gpurun_out/r02_exit_n$N.txt
done; done
for E in poll push; do
  FC_EXIT=$E timeout 600 $TR --master-port 29543 bench.py --gpus $N --steps 200 --warmup 20 --no-baselines --no-cpu-baseline > gpurun_out/r02_exit_bench_${E}_n$N.json 2>/dev/null
  echo "$E bench $(python -c "import json;d=json.load(open('gpurun_out/r02_exit_bench_${E}_n$N.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'])")" >> gpurun_out/r02_exit_n$N.txt
done
timeout 1200 python -m pytest tests/test_multi_gpu.py -x -q -m gpu -k "one_gpu" > gpurun_out/r02_pytest_onegpu.log 2>&1
echo "one-gpu pytest exit=$?" >> gpurun_out/r02_exit_n$N.txt
echo done
