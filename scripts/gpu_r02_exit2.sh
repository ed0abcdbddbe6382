# usage: bash scripts/gpu_r02_exit2.sh   (under gpurun --gpus 4): exit protocol push (rank-level, remote stamps) vs
# ctapoll (per-CTA fence.sys + local stamps polled over NVLink), parity first, then A/B at p = 2 and 4
O=gpurun_out/r02_exit2; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  FC_EXIT=ctapoll FC_MP_TIMEOUT=5 FC_MP_TIMEOUT_TEST=1 FC_MP_STRESS=400 timeout 900 $TR --nproc-per-node $N --master-port 2957$N tests/mp_worker.py > $O/mp_ctapoll_n$N.log 2>&1
  echo "N=$N ctapoll parity rc=$? ok=$(grep -o 'MP_OK' $O/mp_ctapoll_n$N.log | wc -l)" >> $O/summary.txt
done
for N in 4 2; do for rep in 1 2; do for E in push ctapoll; do
  FC_EXIT=$E timeout 300 $TR --nproc-per-node $N --master-port 29581 scripts/gap_coll.py --size 7600000 --dump 2>/dev/null | grep '"fused"' | sed "s/^/N=$N $E rep$rep /" >> $O/gap.txt
  for c in nin googlenet alexnet; do
    FC_EXIT=$E timeout 600 $TR --nproc-per-node $N --master-port 29582 bench.py --gpus $N --config $c --steps 100 --warmup 10 --no-baselines --no-cpu-baseline > $O/b.json 2>/dev/null
    echo "N=$N $E rep$rep $c $(python -c "import json;d=json.load(open('$O/b.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'], all(v if isinstance(v,bool) else v['within_1e-6_of_f64'] for v in d['parity']['executors'].values()))")" >> $O/summary.txt
  done
done; done; done
timeout 900 $TR --nproc-per-node 4 --master-port 29583 examples/nin_dp_torchrun.py --steps 20 > $O/nin_dp_n4.json 2> $O/nin_dp_n4.err
FC_EXIT=ctapoll timeout 900 $TR --nproc-per-node 4 --master-port 29584 examples/nin_dp_torchrun.py --steps 20 > $O/nin_dp_n4_ctapoll.json 2> $O/nin_dp_n4_ctapoll.err
timeout 900 python -m pytest tests/test_multi_gpu.py -q -m gpu -x -k "one_gpu or other_kernel_builds" > $O/pytest_mgpu.log 2>&1; echo "exit $?" >> $O/pytest_mgpu.log
echo done
