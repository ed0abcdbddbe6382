# usage: bash scripts/gpu_tree_lb.sh  — tree-kernel register budgets (FC_TREE_CTAS_PER_SM=2: 128 regs, spills,
# 2 CTAs/SM; =1: spill-free, 1 CTA/SM) at p = 2, 4, and the FLAT unroll at p = 7, 8 on a virtual world
# (profiles/r01_sweep_tree_launch_bounds_*, r01_virtual_flat_unroll_p7_p8.jsonl)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for C in 2 1; do
  for p in 2 4; do
    FC_TREE_CTAS_PER_SM=$C timeout 600 $TR --nproc-per-node $p --master-port $((29600 + p)) scripts/sweep.py \
      --sizes 1048576,7600000,60965224 --scheds forest/direct,forest/tree,single_root/tree,flat/direct \
      > gpurun_out/tree_lb_c${C}_p$p.jsonl 2> gpurun_out/tree_lb_c${C}_p$p.err
  done
done
for p in 7 8; do for u in 1 2 4; do for c in nin alexnet; do
  FC_FLAT_UNROLL=$u timeout 300 python scripts/virtual_time.py $p flat/direct $c
done; done; done > gpurun_out/virt_unroll.jsonl 2> gpurun_out/virt_unroll.err
