# usage: bash scripts/gpu_exit3.sh — rank-level exit: non-last CTAs fence at gpu scope (default) vs sys scope
# (the FC_EXIT variant measured here was not kept in the library; this script is the record of the experiment)
# (FC_EXIT=rank_sys), p = 2, 4, A/B twice, with the one-clock launch/completion breakdown
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for p in 2 4; do
  FC_EXIT=rank_sys FC_MP_TIMEOUT=5 FC_MP_TIMEOUT_TEST=0 timeout 600 $TR --nproc-per-node $p --master-port $((29660 + p)) tests/mp_worker.py \
    > gpurun_out/exit3_mp_p$p.log 2>&1; echo "mp p=$p rc=$? $(grep -o 'MP_OK [0-9]' gpurun_out/exit3_mp_p$p.log | wc -l) ok"
done
for rep in 1 2; do
  for E in rank rank_sys; do
    for p in 2 4; do
      FC_EXIT=$E timeout 600 $TR --nproc-per-node $p --master-port $((29670 + p)) scripts/sweep.py \
        --sizes 65536,1048576,7600000,60965224 --scheds flat/direct --ops fused \
        > gpurun_out/exit3_${E}_p${p}_$rep.jsonl 2> gpurun_out/exit3_${E}_p${p}_$rep.err
      FC_EXIT=$E timeout 200 $TR --nproc-per-node $p --master-port 2959$p scripts/gap_coll.py --size 7600000 2>/dev/null | grep '"fused"' | sed "s/^/$E rep$rep /" >> gpurun_out/exit3_gap.txt
    done
  done
done
