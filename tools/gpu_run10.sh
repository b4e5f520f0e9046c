cd $GRAFT_REPO_ROOT
O=gpurun_out/r10; mkdir -p $O
timeout 900 python -m pytest tests/test_spgemm_gpu.py tests/test_multiproc_gpu.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for cl in 1 8; do
RDMM_SPGEMM_CL=$cl timeout 300 python tools/spgemm_time.py --scale 17 > $O/sg17_cl$cl.json 2>&1
RDMM_SPGEMM_CL=$cl timeout 300 python tools/spgemm_time.py --scale 20 > $O/sg20_cl$cl.json 2>&1
done
timeout 300 python tools/spgemm_time.py --scale 20 --iters 1 > $O/plain_sg.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_spgemm20.csv python tools/spgemm_time.py --scale 20 --iters 1 > $O/ncu_sg.log 2>&1
echo finished
