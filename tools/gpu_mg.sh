# usage: bash tools/gpu_mg.sh NGPUS
N=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/mg$N; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531"
timeout 600 $T bench.py --gpus $N --steps 10 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 $T bench.py --gpus $N --steps 10 --variant summa_nccl > $O/bench_cfg3_summa.json 2> $O/bench_cfg3_summa.err
timeout 600 $T bench.py --gpus $N --steps 10 --variant ws_locality > $O/bench_cfg3_wsl.json 2> $O/bench_cfg3_wsl.err
if [ "$N" = "4" ]; then timeout 600 $T bench.py --gpus $N --steps 10 --grid 2x2 > $O/bench_cfg3_2x2.json 2> $O/bench_cfg3_2x2.err; fi
timeout 600 $T bench.py --gpus $N --steps 10 --config cfg5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 $T bench.py --gpus $N --steps 3 --config cfg4 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 $T bench.py --gpus $N --steps 3 --config cfg2 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
du -sh $O
echo finished
