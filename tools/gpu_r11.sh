# usage: bash tools/gpu_r11.sh (1 GPU): SpGEMM s20 launch list after the dense-tier changes
cd $GRAFT_REPO_ROOT
O=gpurun_out/r11; mkdir -p $O
timeout 600 python tools/spgemm_time.py --scale 20 --iters 1 > $O/sg20.json 2> $O/sg20.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/sg20_launches.csv python tools/spgemm_time.py --scale 20 --iters 1 > $O/ncu.log 2>&1
echo finished
