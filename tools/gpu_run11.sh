cd $GRAFT_REPO_ROOT
O=gpurun_out/r11; mkdir -p $O
timeout 300 python tools/spgemm_time.py --scale 17 --iters 1 > $O/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_num -c 1 -o $O/prof_dense17 python tools/spgemm_time.py --scale 17 --iters 1 > $O/ncu.log 2>&1
ls -la $O
echo finished
