# usage: bash tools/gpu_r3a.sh (1 GPU): concat tests + hint sweep + 1-GPU bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3; mkdir -p $O
timeout 600 python -m pytest tests/test_util_gpu.py tests/test_algos_gpu.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
bash tools/gpu_hint.sh
timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/b1_cfg3.json 2> $O/b1_cfg3.err
echo finished
