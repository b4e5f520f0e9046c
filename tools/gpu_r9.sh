# usage: bash tools/gpu_r9.sh (1 GPU): SpGEMM flat vs warp enumeration (+ load-before-CAS)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r9; mkdir -p $O
for f in 0 1; do
  RDMM_SPGEMM_FLAT=$f timeout 300 python tools/spgemm_time.py --scale 17 > $O/sg17_f$f.json 2> $O/sg17_f$f.err
  RDMM_SPGEMM_FLAT=$f timeout 600 python tools/spgemm_time.py --scale 20 --iters 2 > $O/sg20_f$f.json 2> $O/sg20_f$f.err
done
RDMM_SPGEMM_FLAT=1 timeout 900 python -m pytest tests/test_spgemm_gpu.py -x -q > $O/pytest_f1.log 2>&1; echo "pytest rc=$?" >> $O/pytest_f1.log
timeout 900 python -m pytest tests/test_spgemm_gpu.py -x -q > $O/pytest_f0.log 2>&1; echo "pytest rc=$?" >> $O/pytest_f0.log
echo finished
