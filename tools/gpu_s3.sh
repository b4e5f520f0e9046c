# session-2 check with the model block: 1-GPU cfg3/cfg4, 2-GPU cfg3/cfg5
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563"
timeout 600 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 python bench.py --config cfg4 --steps 3 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 600 $T bench.py --gpus 2 --steps 10 > $O/bench2_cfg3.json 2> $O/bench2_cfg3.err
timeout 600 $T bench.py --gpus 2 --steps 10 --config cfg5 --no-cpu-baseline > $O/bench2_cfg5.json 2> $O/bench2_cfg5.err
timeout 900 $T bench.py --gpus 2 --impl reference --steps 2 > $O/ref2_cfg3.json 2> $O/ref2_cfg3.err
echo finished
