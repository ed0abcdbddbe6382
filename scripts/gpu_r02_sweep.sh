# usage: bash scripts/gpu_r02_sweep.sh  (under gpurun --gpus 4): size x executor sweep of the final build at p = 2, 4
# (fused; every executor + PS + NCCL, phase traces) for the f1 table/calibration, and five f3 overlap runs at p = 2
O=gpurun_out/r02_sweep; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 1500 $TR --nproc-per-node $N --master-port 2968$N scripts/sweep.py --sizes 65536,1048576,4194304,7600000,13250000,60965224 \
    --ops fused,ps --nccl --iters 30 2>/dev/null | grep '^{' > $O/sweep_p$N.jsonl
done
for run in 1 2 3 4 5; do
  timeout 900 $TR --nproc-per-node 2 --master-port 29689 examples/nin_dp_torchrun.py --steps 20 2>/dev/null | grep '^{' >> $O/nin_dp_overlap_n2.jsonl
done
echo done
