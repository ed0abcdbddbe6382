# usage: bash scripts/gpu_flat_db.sh — FLAT single- vs register double-buffered (FC_FLAT_DB), p = 2, 4; parity first
# (FC_FLAT_DB selected a register double-buffered FLAT build that was measured, not adopted and removed; kept as the record of the experiment)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "every_kernel_build and FC_FLAT_DB" > gpurun_out/flatdb_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/flatdb_pytest.log
for p in 2 4; do
  FC_FLAT_DB=1 FC_MP_TIMEOUT=5 timeout 600 $TR --nproc-per-node $p --master-port $((29660 + p)) tests/mp_worker.py \
    > gpurun_out/flatdb_mp_p$p.log 2>&1; echo "mp p=$p rc=$? $(grep -c MP_OK gpurun_out/flatdb_mp_p$p.log) ok"
done
for rep in 1 2; do
  for D in 0 1; do
    for p in 2 4; do
      FC_FLAT_DB=$D timeout 600 $TR --nproc-per-node $p --master-port $((29670 + p)) scripts/sweep.py \
        --sizes 65536,1048576,7600000,13250000,60965224 --scheds flat/direct --ops fused \
        > gpurun_out/flatdb_${D}_p${p}_$rep.jsonl 2> gpurun_out/flatdb_${D}_p${p}_$rep.err
    done
  done
done
