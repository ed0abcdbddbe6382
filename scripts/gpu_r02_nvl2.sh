# usage: bash scripts/gpu_r02_nvl2.sh  (under gpurun --gpus 2): NVLink bytes of one fused FLAT launch on rank 0 of a
# real 2-GPU world (rank 0 under ncu with a single-pass metric set, rank 1 plain)
O=gpurun_out/r02_nvl2; mkdir -p $O
for c in nin alexnet; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 \
    --no-python scripts/ncu_rank0.sh $O/nvl_$c.csv scripts/real_flat_run.py $c > $O/nvl_$c.log 2>&1
  echo "$c exit $?" >> $O/nvl_$c.log
done
echo done
