# usage: bash tools/gpu_r13.sh (1 GPU): SpMM stream kernel with the window loop not unrolled; SpGEMM restored
cd $GRAFT_REPO_ROOT
O=gpurun_out/r13; mkdir -p $O
S="timeout 300 python tools/spmm_time.py --czero 1 --iters 20"
$S --tag rolled > $O/spmm.jsonl 2> $O/spmm.err
$S --tag rolled_er --er >> $O/spmm.jsonl 2>> $O/spmm.err
timeout 300 python tools/spmm_time.py --czero 1 --iters 20 --scale 16 --ef 8 --tag rolled_s16 >> $O/spmm.jsonl 2>> $O/spmm.err
timeout 600 python tools/spgemm_time.py --scale 20 --iters 2 > $O/sg20.json 2> $O/sg20.err
timeout 900 python -m pytest tests/test_spmm_gpu.py tests/test_spgemm_gpu.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
echo finished
