# usage: bash tools/gpu_r10.sh (1 GPU): SpGEMM with the 4-way write-combining cache
cd $GRAFT_REPO_ROOT
O=gpurun_out/r12; mkdir -p $O
timeout 300 python tools/spgemm_time.py --scale 17 > $O/sg17.json 2> $O/sg17.err
timeout 600 python tools/spgemm_time.py --scale 20 --iters 2 > $O/sg20.json 2> $O/sg20.err
timeout 900 python -m pytest tests/test_spgemm_gpu.py tests/test_algos_gpu.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 3 --config cfg4 --no-cpu-baseline > $O/b1_cfg4.json 2> $O/b1_cfg4.err
timeout 600 python bench.py --steps 5 --config cfg2 --no-cpu-baseline > $O/b1_cfg2.json 2> $O/b1_cfg2.err
echo finished
