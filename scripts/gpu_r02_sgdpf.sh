# usage: bash scripts/gpu_r02_sgdpf.sh (under gpurun, 1 GPU): 1-GPU SGD loads with the L2::256B hint (FC_SGD_PF=256) vs
# plain, A/B three times at every config size; parity of the hinted build
O=gpurun_out/r02_sgdpf; mkdir -p $O
FC_SGD_PF=256 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "sgd_step_bitexact or full_nin_size or beyond_2_31_elements and not virtual" > $O/pytest.log 2>&1; echo "parity(pf) exit $?" >> $O/summary.txt
for rep in 1 2 3; do for PF in 256 0; do for c in nin googlenet alexnet vgg19; do
  FC_SGD_PF=$PF timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-baselines --no-cpu-baseline --no-steady > $O/b.json 2>/dev/null
  echo "pf=$PF rep$rep $c $(python -c "import json;d=json.load(open('$O/b.json'));print(d['ms_per_step'], d['roofline']['frac'], d['parity']['bitexact_sampled'])")" >> $O/summary.txt
done; done; done
echo done
