cd $GRAFT_REPO_ROOT
O=gpurun_out/r8; mkdir -p $O
timeout 600 python bench.py --steps 10 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --steps 10 --config cfg5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 300 python tools/spgemm_time.py --scale 20 --iters 1 > $O/plain_sg.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_spgemm20.csv python tools/spgemm_time.py --scale 20 --iters 1 > $O/ncu_sg.log 2>&1
echo finished
