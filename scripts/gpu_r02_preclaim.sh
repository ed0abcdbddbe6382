# usage: bash scripts/gpu_r02_preclaim.sh  (under gpurun --gpus 4): FLAT first claim before the entry barrier (default)
# vs after it (FC_FLAT_PRECLAIM=0); parity first; A/B twice at p = 4, 2 (NiN, GoogLeNet)
O=gpurun_out/r02_preclaim; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  FC_MP_TIMEOUT=5 FC_MP_STRESS=400 timeout 900 $TR --nproc-per-node $N --master-port 2966$N tests/mp_worker.py > $O/mp_n$N.log 2>&1
  echo "N=$N parity rc=$? ok=$(grep -o 'MP_OK' $O/mp_n$N.log | wc -l)" >> $O/summary.txt
done
for N in 4 2; do for rep in 1 2 3; do for PC in 1 0; do for c in nin googlenet; do
  FC_FLAT_PRECLAIM=$PC timeout 600 $TR --nproc-per-node $N --master-port 29665 bench.py --gpus $N --config $c --steps 200 --warmup 10 --no-baselines --no-cpu-baseline > $O/b.json 2>/dev/null
  echo "N=$N preclaim=$PC rep$rep $c $(python -c "import json;d=json.load(open('$O/b.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'], all(v if isinstance(v,bool) else v['within_1e-6_of_f64'] for v in d['parity']['executors'].values()))")" >> $O/summary.txt
done; done; done; done
echo done
