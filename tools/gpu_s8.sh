# cfg2 with its new default (stationary_c, square-ish grid) at 1 / 2 / 4 GPUs
cd $GRAFT_REPO_ROOT
O=gpurun_out/s8; mkdir -p $O
timeout 600 python bench.py --config cfg2 --steps 5 --no-cpu-baseline > $O/cfg2_1.json 2> $O/cfg2_1.err
for N in 2 4; do
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N"
  timeout 600 $T bench.py --gpus $N --steps 5 --config cfg2 --no-cpu-baseline > $O/cfg2_$N.json 2> $O/cfg2_$N.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29589 bench.py --gpus 4 --steps 5 --config cfg2 --variant stationary_a --no-cpu-baseline > $O/cfg2_4_sa.json 2> $O/cfg2_4_sa.err
echo finished
