# usage: bash scripts/gpu_exit_sweep.sh  — per-CTA vs rank-level exit protocol (FC_EXIT) at p = 2, 4
# (profiles/r01_sweep_exit_*.jsonl); real-world parity under FC_EXIT=rank first
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for p in 2 4; do
  FC_EXIT=rank FC_MP_TIMEOUT=5 timeout 600 $TR --nproc-per-node $p --master-port $((29660 + p)) tests/mp_worker.py \
    > gpurun_out/exit_mp_p$p.log 2>&1; echo "mp p=$p rc=$? $(grep -c MP_OK gpurun_out/exit_mp_p$p.log) ok"
done
for E in cta rank; do
  for p in 2 4; do
    FC_EXIT=$E timeout 900 $TR --nproc-per-node $p --master-port $((29670 + p)) scripts/sweep.py \
      --sizes 65536,1048576,7600000,13250000,60965224 --scheds flat/direct,forest/direct,single_root/direct \
      --ops fused,allreduce > gpurun_out/exit_${E}_p$p.jsonl 2> gpurun_out/exit_${E}_p$p.err
  done
done
