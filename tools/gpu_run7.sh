cd $GRAFT_REPO_ROOT
O=gpurun_out/r7; mkdir -p $O
RDMM_TRACE=1 timeout 600 python bench.py --steps 4 --no-cpu-baseline > $O/bench_trace.json 2> $O/bench_trace.err
timeout 600 python bench.py --steps 10 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
echo finished
