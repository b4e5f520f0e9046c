cd $GRAFT_REPO_ROOT
O=gpurun_out/r14; mkdir -p $O
timeout 900 python -m pytest tests/test_spmm_gpu.py tests/test_spgemm_gpu.py tests/test_algos_gpu.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for n in 8 16 32 64 128; do
  timeout 120 python tools/spmm_time.py --n $n --czero 1 --tag "n$n auto" >> $O/sweep.jsonl 2>>$O/sweep.err
done
for n in 16 32 64; do
  RDMM_SPMM_KERNEL=rows timeout 120 python tools/spmm_time.py --n $n --czero 1 --tag "n$n rows" >> $O/sweep.jsonl 2>>$O/sweep.err
done
timeout 300 python bench.py --steps 10 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 300 python tools/spgemm_time.py --scale 17 > $O/sg17.json 2>&1
timeout 300 python tools/spgemm_time.py --scale 20 > $O/sg20.json 2>&1
echo finished
