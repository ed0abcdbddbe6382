# usage: bash scripts/gpu_sweep.sh N [tag] [extra sweep args...]
N=${1:-2}; TAG=${2:-x}; shift 2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513"
timeout 900 $TR scripts/sweep.py "$@" > gpurun_out/sweep_${TAG}_n$N.jsonl 2> gpurun_out/sweep_${TAG}_n$N.err
