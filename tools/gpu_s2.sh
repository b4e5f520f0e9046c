# session-2 check on 2 GPUs: gpu tests, smoke, 1-GPU cfg3 bench, 2-GPU cfg3/cfg2 with stage imbalance
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562"
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 $T bench.py --gpus 2 --steps 10 > $O/bench2_cfg3.json 2> $O/bench2_cfg3.err
timeout 600 $T bench.py --gpus 2 --steps 5 --config cfg2 --no-cpu-baseline > $O/bench2_cfg2.json 2> $O/bench2_cfg2.err
echo finished
