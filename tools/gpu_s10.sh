# cfg4 / cfg2 default (square grid) confirmation at 2 and 4 GPUs; ws_random with its stationary_a base
cd $GRAFT_REPO_ROOT
O=gpurun_out/s10; mkdir -p $O
for N in 4 2; do
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N"
  timeout 600 $T bench.py --gpus $N --steps 3 --config cfg4 --no-cpu-baseline > $O/cfg4_$N.json 2> $O/cfg4_$N.err
done
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29609"
timeout 600 $T bench.py --gpus 4 --steps 3 --config cfg4 --variant ws_random --no-cpu-baseline > $O/cfg4_4_wsr.json 2> $O/cfg4_4_wsr.err
timeout 600 $T bench.py --gpus 4 --steps 3 --config cfg4 --permute 7 --no-cpu-baseline > $O/cfg4_4_perm.json 2> $O/cfg4_4_perm.err
echo finished
