# usage: bash scripts/gpu_exit2.sh  — rank-level exit: parallel st.release.sys (FC_EXIT=rank, default)
# vs one fence.sys + relaxed stamps (FC_EXIT=rank_fence), p = 2, 4, A/B/A/B; parity first
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for p in 2 4; do
  FC_MP_TIMEOUT=5 timeout 600 $TR --nproc-per-node $p --master-port $((29660 + p)) tests/mp_worker.py \
    > gpurun_out/exit2_mp_p$p.log 2>&1; echo "mp p=$p rc=$? $(grep -c MP_OK gpurun_out/exit2_mp_p$p.log) ok"
done
for rep in 1 2; do
  for E in rank rank_fence; do
    for p in 2 4; do
      FC_EXIT=$E timeout 600 $TR --nproc-per-node $p --master-port $((29670 + p)) scripts/sweep.py \
        --sizes 65536,1048576,7600000,60965224 --scheds flat/direct,forest/direct --ops fused \
        > gpurun_out/exit2_${E}_p${p}_$rep.jsonl 2> gpurun_out/exit2_${E}_p${p}_$rep.err
    done
  done
done
for p in 2 4; do
  timeout 600 $TR --nproc-per-node $p --master-port 29514 bench.py --gpus $p --no-baselines > gpurun_out/exit2_bench_n$p.json 2> gpurun_out/exit2_bench_n$p.err
done
