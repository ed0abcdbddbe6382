# usage: bash scripts/gpu_r02_clean.sh  (under gpurun --gpus 4): rank-level exit with the non-last CTAs fencing at sys
# scope after arriving (FC_CLEAN_EXIT=1) vs leaving at once (default); parity first; A/B three times at p = 4, 2;
# one-clock breakdown (completion) at NiN p = 4
O=gpurun_out/r02_clean; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  FC_CLEAN_EXIT=1 FC_MP_TIMEOUT=5 FC_MP_STRESS=400 timeout 900 $TR --nproc-per-node $N --master-port 2971$N tests/mp_worker.py > $O/mp_n$N.log 2>&1
  echo "N=$N parity(clean) rc=$? ok=$(grep -o 'MP_OK' $O/mp_n$N.log | wc -l)" >> $O/summary.txt
done
for N in 4 2; do for rep in 1 2 3; do for E in 1 0; do for c in nin googlenet alexnet; do
  FC_CLEAN_EXIT=$E timeout 600 $TR --nproc-per-node $N --master-port 29715 bench.py --gpus $N --config $c --steps 200 --warmup 10 --no-baselines --no-cpu-baseline > $O/b.json 2>/dev/null
  echo "N=$N clean=$E rep$rep $c $(python -c "import json;d=json.load(open('$O/b.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'], all(v if isinstance(v,bool) else v['within_1e-6_of_f64'] for v in d['parity']['executors'].values()))")" >> $O/summary.txt
done; done; done; done
for E in 1 0; do FC_CLEAN_EXIT=$E timeout 300 $TR --nproc-per-node 4 --master-port 29716 scripts/gap_coll.py --size 7600000 2>/dev/null | grep '"fused"' | sed "s/^/clean=$E /" >> $O/gap_n4.txt; done
echo done
