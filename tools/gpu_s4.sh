# session-2: gpu tests (permute_symmetric, stage flops), permuted R-MAT SpMM / SpGEMM at 1 and 2 GPUs
cd $GRAFT_REPO_ROOT
O=gpurun_out/s4; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29564"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --permute 7 --no-cpu-baseline > $O/bench_cfg3_perm.json 2> $O/bench_cfg3_perm.err
timeout 600 $T bench.py --gpus 2 --steps 10 --permute 7 --no-cpu-baseline > $O/bench2_cfg3_perm.json 2> $O/bench2_cfg3_perm.err
timeout 900 python bench.py --config cfg4 --steps 3 --permute 7 --no-cpu-baseline > $O/bench_cfg4_perm.json 2> $O/bench_cfg4_perm.err
timeout 900 $T bench.py --gpus 2 --steps 3 --config cfg4 --permute 7 --no-cpu-baseline > $O/bench2_cfg4_perm.json 2> $O/bench2_cfg4_perm.err
echo finished
