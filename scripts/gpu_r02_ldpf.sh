# usage: bash scripts/gpu_r02_ldpf.sh  (under gpurun --gpus 4): FLAT operand loads with the L2::256B prefetch-size hint
# (FC_LD_PF=256) vs plain; parity first; A/B twice at p = 4, 2 (NiN, GoogLeNet, AlexNet)
O=gpurun_out/r02_ldpf; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  FC_LD_PF=256 FC_MP_TIMEOUT=5 FC_MP_STRESS=300 timeout 900 $TR --nproc-per-node $N --master-port 2969$N tests/mp_worker.py > $O/mp_n$N.log 2>&1
  echo "N=$N parity(pf256) rc=$? ok=$(grep -o 'MP_OK' $O/mp_n$N.log | wc -l)" >> $O/summary.txt
done
for N in 4 2; do for rep in 1 2; do for PF in 256 0; do for c in nin googlenet alexnet; do
  FC_LD_PF=$PF timeout 600 $TR --nproc-per-node $N --master-port 29695 bench.py --gpus $N --config $c --steps 100 --warmup 10 --no-baselines --no-cpu-baseline > $O/b.json 2>/dev/null
  echo "N=$N pf=$PF rep$rep $c $(python -c "import json;d=json.load(open('$O/b.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'])")" >> $O/summary.txt
done; done; done; done
echo done
