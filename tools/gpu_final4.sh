cd $GRAFT_REPO_ROOT
O=gpurun_out/f4; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1; nproc > $O/nproc.txt
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for c in cfg1 cfg5 cfg2 cfg4; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py --variant summa_nccl --no-cpu-baseline > $O/bench_cfg3_summa.json 2> $O/bench_cfg3_summa.err
timeout 900 python bench.py --impl reference > $O/ref_cfg3.json 2> $O/ref_cfg3.err
timeout 900 python bench.py --impl reference --config cfg4 --steps 2 > $O/ref_cfg4.json 2> $O/ref_cfg4.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
ls -la $O; du -sh $O
echo finished
