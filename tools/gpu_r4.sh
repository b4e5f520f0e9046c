# usage: bash tools/gpu_r4.sh (1 GPU): SpGEMM tier breakdown + per-kernel launch times
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4; mkdir -p $O
timeout 300 python tools/spgemm_time.py --scale 17 > $O/sg17.json 2> $O/sg17.err
timeout 600 python tools/spgemm_time.py --scale 20 --iters 2 > $O/sg20.json 2> $O/sg20.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/sg20_launches.csv python tools/spgemm_time.py --scale 20 --iters 1 > $O/ncu.log 2>&1
echo finished
