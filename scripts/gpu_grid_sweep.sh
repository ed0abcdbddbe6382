# usage: bash scripts/gpu_grid_sweep.sh  — FLAT grid size vs message size at p = 2, 4 (profiles/r01_sweep_flat_grid_p*.jsonl)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for p in 2 4; do
  timeout 900 $TR --nproc-per-node $p --master-port $((29640 + p)) scripts/sweep.py --sizes 65536,1048576,4194304,7600000,13250000 \
    --scheds flat/direct --max-ctas 16,32,64,96,128,0 > gpurun_out/grid_p$p.jsonl 2> gpurun_out/grid_p$p.err
done
