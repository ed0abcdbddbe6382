# usage: bash scripts/gpu_flat_map.sh — FLAT work mapping: balanced slab rows (default) vs plain grid stride
# (FC_FLAT_MAP=stride), p = 2, 4, A/B twice; parity first (virtual worlds + real 2/4-GPU worlds)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "virtual_fused or virtual_tree_allreduce or virtual_ps or back_to_back or capped_grid or host" > gpurun_out/map_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/map_pytest.log
for p in 2 4; do
  FC_MP_TIMEOUT=5 timeout 600 $TR --nproc-per-node $p --master-port $((29660 + p)) tests/mp_worker.py \
    > gpurun_out/map_mp_p$p.log 2>&1; echo "mp p=$p rc=$? $(grep -o 'MP_OK [0-9]' gpurun_out/map_mp_p$p.log | wc -l) ok"
done
for rep in 1 2; do
  for M in balanced stride; do
    for p in 2 4; do
      FC_FLAT_MAP=$M timeout 600 $TR --nproc-per-node $p --master-port $((29670 + p)) scripts/sweep.py \
        --sizes 65536,1048576,7600000,13250000,60965224 --scheds flat/direct --ops fused,allreduce \
        > gpurun_out/map_${M}_p${p}_$rep.jsonl 2> gpurun_out/map_${M}_p${p}_$rep.err
    done
  done
done
for p in 2 4; do
  timeout 200 $TR --nproc-per-node $p --master-port 2959$p scripts/gap_coll.py --size 7600000 2>/dev/null | grep fused > gpurun_out/map_gap_p$p.jsonl
done
