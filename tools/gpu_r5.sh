# usage: bash tools/gpu_r5.sh (1 GPU): fused stationary-C (K=2 on one GPU) + its launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/r5; mkdir -p $O
timeout 300 python bench.py --steps 5 --ktiles 2 --no-cpu-baseline > $O/k2.json 2> $O/k2.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/k2_launches.csv python bench.py --steps 2 --warmup 3 --ktiles 2 --no-cpu-baseline > $O/ncu.log 2>&1
echo finished
