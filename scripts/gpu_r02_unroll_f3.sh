# usage: bash scripts/gpu_r02_unroll_f3.sh   (under gpurun --gpus 4): FLAT unroll with the dynamic claims (p=2: U=4 vs 2,
# p=4: U=2 vs 1; A/B twice) and five runs of the f3 overlap measurement at p = 4
O=gpurun_out/r02_uf3; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for rep in 1 2; do
  for U in 4 2; do FC_FLAT_UNROLL=$U timeout 600 $TR --nproc-per-node 2 --master-port 29601 scripts/sweep.py --sizes 7600000,13250000,60965224 --scheds flat/direct --iters 30 2>/dev/null | sed "s/^/U=$U rep$rep /" >> $O/unroll.txt; done
  for U in 2 1; do FC_FLAT_UNROLL=$U timeout 600 $TR --nproc-per-node 4 --master-port 29602 scripts/sweep.py --sizes 7600000,13250000,60965224 --scheds flat/direct --iters 30 2>/dev/null | sed "s/^/U=$U rep$rep /" >> $O/unroll.txt; done
done
for run in 1 2 3 4 5; do
  timeout 900 $TR --nproc-per-node 4 --master-port 29603 examples/nin_dp_torchrun.py --steps 20 2>/dev/null | grep '^{' >> $O/nin_dp_overlap_n4.jsonl
done
echo done
