# usage: bash scripts/gpu_exit4.sh — counted exit (FC_EXIT=count: per-CTA sys fence + counter adds into
# (the FC_EXIT variant measured here was not kept in the library; this script is the record of the experiment)
# the peers, the last CTA waits for the peers' counts) vs the rank-level exit (default), p = 2, 4, A/B twice;
# parity first (real 2/4-GPU worlds incl. stress, virtual worlds)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_gpu_parity.py -q -x -k "count" > gpurun_out/exit4_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/exit4_pytest.log
for rep in 1 2; do
  for E in rank count; do
    for p in 2 4; do
      FC_EXIT=$E timeout 600 $TR --nproc-per-node $p --master-port $((29670 + p)) scripts/sweep.py \
        --sizes 65536,1048576,7600000,13250000,60965224 --scheds flat/direct,forest/direct --ops fused,allreduce \
        > gpurun_out/exit4_${E}_p${p}_$rep.jsonl 2> gpurun_out/exit4_${E}_p${p}_$rep.err
      FC_EXIT=$E timeout 200 $TR --nproc-per-node $p --master-port 2959$p scripts/gap_coll.py --size 7600000 2>/dev/null | grep '"fused"' | sed "s/^/$E rep$rep /" >> gpurun_out/exit4_gap.txt
    done
  done
done
