# usage: bash tools/gpu_hint.sh  (1 GPU): L2 residency hint sweep on cfg3 / cfg5
cd $GRAFT_REPO_ROOT
O=gpurun_out/hint; mkdir -p $O
S="timeout 300 python tools/spmm_time.py --czero 1 --iters 20"
$S --tag base > $O/sweep.jsonl 2> $O/sweep.err
for m in 1 2 3; do RDMM_SPMM_L2HINT=$m $S --tag m$m >> $O/sweep.jsonl 2>> $O/sweep.err; done
for mb in 32 96 128 160; do RDMM_SPMM_L2HINT=1 RDMM_SPMM_L2HOT_MB=$mb $S --tag m1_$mb >> $O/sweep.jsonl 2>> $O/sweep.err; done
for mb in 32 96 128; do RDMM_SPMM_L2HINT=2 RDMM_SPMM_L2HOT_MB=$mb $S --tag m2_$mb >> $O/sweep.jsonl 2>> $O/sweep.err; done
$S --tag base_er --er > $O/sweep_er.jsonl 2>> $O/sweep.err
RDMM_SPMM_L2HINT=1 $S --tag m1_er --er >> $O/sweep_er.jsonl 2>> $O/sweep.err
RDMM_SPMM_L2HINT=1 timeout 900 python -m pytest tests/test_spmm_gpu.py -x -q > $O/pytest_hint.log 2>&1; echo "rc=$?" >> $O/pytest_hint.log
echo finished
