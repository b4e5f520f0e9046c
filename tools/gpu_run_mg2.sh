cd $GRAFT_REPO_ROOT
O=gpurun_out/mg2; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 600 python -m pytest tests/test_multiproc_gpu.py -x -q > $O/pytest_mp.log 2>&1; echo "rc=$?" >> $O/pytest_mp.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
timeout 600 $T bench.py --gpus 2 --steps 10 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 $T bench.py --gpus 2 --steps 10 --variant summa_nccl > $O/bench_cfg3_summa.json 2> $O/bench_cfg3_summa.err
timeout 600 $T bench.py --gpus 2 --steps 10 --variant ws_locality > $O/bench_cfg3_wsl.json 2> $O/bench_cfg3_wsl.err
timeout 600 $T bench.py --gpus 2 --steps 10 --grid 2x1 > $O/bench_cfg3_2x1.json 2> $O/bench_cfg3_2x1.err
timeout 900 $T bench.py --gpus 2 --steps 3 --config cfg4 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
echo finished
