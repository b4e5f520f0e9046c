cd $GRAFT_REPO_ROOT
O=gpurun_out/r5; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for c in cfg1 cfg5 cfg2 cfg4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py --variant ws_locality --no-cpu-baseline > $O/bench_cfg3_wsl.json 2> $O/bench_cfg3_wsl.err
timeout 600 python bench.py --variant summa_nccl --no-cpu-baseline > $O/bench_cfg3_summa.json 2> $O/bench_cfg3_summa.err
timeout 900 python bench.py --impl reference > $O/ref_cfg3.json 2> $O/ref_cfg3.err
echo finished
