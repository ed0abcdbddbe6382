# usage: bash scripts/gpu_r02_quarter.sh  (under gpurun --gpus 4): FLAT dynamic claims in quarter units (dyn, new default)
# vs whole units (dyn1), parity first, A/B twice at p = 2, 4 (NiN, GoogLeNet, AlexNet), one-clock breakdown at NiN p=4
O=gpurun_out/r02_quarter; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  FC_MP_TIMEOUT=5 FC_MP_STRESS=400 timeout 900 $TR --nproc-per-node $N --master-port 2964$N tests/mp_worker.py > $O/mp_n$N.log 2>&1
  echo "N=$N parity rc=$? ok=$(grep -o 'MP_OK' $O/mp_n$N.log | wc -l)" >> $O/summary.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "virtual_fused_bitexact or virtual_tree_allreduce or virtual_ps or beyond_2_31" > $O/pytest_virtual.log 2>&1; echo "virtual pytest exit $?" >> $O/summary.txt
for N in 4 2; do for rep in 1 2; do for M in dyn dyn1; do for c in nin googlenet alexnet; do
  FC_FLAT_MAP=$M timeout 600 $TR --nproc-per-node $N --master-port 29645 bench.py --gpus $N --config $c --steps 100 --warmup 10 --no-baselines --no-cpu-baseline > $O/b.json 2>/dev/null
  echo "N=$N $M rep$rep $c $(python -c "import json;d=json.load(open('$O/b.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'], all(v if isinstance(v,bool) else v['within_1e-6_of_f64'] for v in d['parity']['executors'].values()))")" >> $O/summary.txt
done; done; done; done
for M in dyn dyn1; do FC_FLAT_MAP=$M timeout 300 $TR --nproc-per-node 4 --master-port 29646 scripts/gap_coll.py --size 7600000 --dump 2>/dev/null | grep '"fused"' | sed "s/^/$M /" >> $O/gap_n4.txt; done
echo done
