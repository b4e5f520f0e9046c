# usage: bash tools/gpu_r8.sh (1 GPU): SpGEMM A/B after the pipelined heavy-row enumeration
cd $GRAFT_REPO_ROOT
O=gpurun_out/r8; mkdir -p $O
timeout 300 python tools/spgemm_time.py --scale 17 > $O/sg17.json 2> $O/sg17.err
timeout 600 python tools/spgemm_time.py --scale 20 --iters 2 > $O/sg20.json 2> $O/sg20.err
timeout 900 python -m pytest tests/test_spgemm_gpu.py tests/test_algos_gpu.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
echo finished
