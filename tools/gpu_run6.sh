cd $GRAFT_REPO_ROOT
O=gpurun_out/r6; mkdir -p $O
timeout 300 python tools/diag_heap.py > $O/diag_heap.log 2>&1
RDMM_TRACE=1 timeout 600 python bench.py --steps 3 --no-cpu-baseline > $O/bench_trace.json 2> $O/bench_trace.err
RDMM_TRACE=1 timeout 600 python bench.py --config cfg2 --steps 2 --no-cpu-baseline > $O/bench_trace2.json 2> $O/bench_trace2.err
timeout 300 python tools/spgemm_time.py --scale 17 > $O/spgemm17.json 2>&1
timeout 300 python tools/spgemm_time.py --scale 20 > $O/spgemm20.json 2>&1
echo finished
