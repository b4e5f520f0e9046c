cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
for occ in 1 4; do for pf in 0 1; do for cz in 0 1; do
  RDMM_SPMM_OCC=$occ RDMM_SPMM_PREFETCH=$pf timeout 120 python tools/spmm_time.py --czero $cz --tag "occ$occ pf$pf cz$cz" >> gpurun_out/sweep2.jsonl 2>>gpurun_out/sweep2.err
done; done; done
for occ in 1 4; do for pf in 0 1; do
  RDMM_SPMM_OCC=$occ RDMM_SPMM_PREFETCH=$pf timeout 120 python tools/spmm_time.py --er --n 256 --czero 1 --tag "er occ$occ pf$pf" >> gpurun_out/sweep2.jsonl 2>>gpurun_out/sweep2.err
done; done
echo finished
