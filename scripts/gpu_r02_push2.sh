# usage: bash scripts/gpu_r02_push2.sh  (under gpurun --gpus 4): rank-level exit push (default) vs push2 (relaxed
# arrival finds the last CTA first, no gpu fence on its critical path); parity first; A/B three times at p = 4, 2
O=gpurun_out/r02_push2; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  FC_EXIT=push2 FC_MP_TIMEOUT=5 FC_MP_STRESS=600 timeout 900 $TR --nproc-per-node $N --master-port 2970$N tests/mp_worker.py > $O/mp_n$N.log 2>&1
  echo "N=$N parity(push2) rc=$? ok=$(grep -o 'MP_OK' $O/mp_n$N.log | wc -l)" >> $O/summary.txt
done
FC_EXIT=push2 FC_MP_GPUS=4 FC_MP_SIZES=5,16391,300007 FC_MP_TIMEOUT=30 FC_MP_TIMEOUT_TEST=0 FC_MP_STRESS=300 timeout 900 $TR --nproc-per-node 8 --master-port 29709 tests/mp_worker.py > $O/mp_8on4.log 2>&1
echo "8on4 parity(push2) rc=$? ok=$(grep -o 'MP_OK' $O/mp_8on4.log | wc -l)" >> $O/summary.txt
FC_EXIT=push2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "virtual_fused_bitexact or virtual_ps or virtual_tree_allreduce" > $O/pytest_virtual.log 2>&1; echo "virtual pytest(push2) exit $?" >> $O/summary.txt
for N in 4 2; do for rep in 1 2 3; do for E in push2 push; do for c in nin googlenet; do
  FC_EXIT=$E timeout 600 $TR --nproc-per-node $N --master-port 29705 bench.py --gpus $N --config $c --steps 200 --warmup 10 --no-baselines --no-cpu-baseline > $O/b.json 2>/dev/null
  echo "N=$N $E rep$rep $c $(python -c "import json;d=json.load(open('$O/b.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'], all(v if isinstance(v,bool) else v['within_1e-6_of_f64'] for v in d['parity']['executors'].values()))")" >> $O/summary.txt
done; done; done; done
for E in push2 push; do FC_EXIT=$E timeout 300 $TR --nproc-per-node 4 --master-port 29706 scripts/gap_coll.py --size 7600000 2>/dev/null | grep '"fused"' | sed "s/^/$E /" >> $O/gap_n4.txt; done
echo done
