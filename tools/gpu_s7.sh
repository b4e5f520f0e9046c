# session-2 final check of the committed tree: gpu tests, smoke, default bench, reference arm, launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/s7; mkdir -p $O
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 python bench.py --impl reference > $O/ref_cfg3.json 2> $O/ref_cfg3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo finished
