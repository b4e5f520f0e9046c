cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r4
O=gpurun_out/r4
timeout 1200 python -m pytest tests -m gpu -x -q -k "not cfg4 and not cfg2" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for k in rows stream; do for occ in 1 4; do for cz in 0 1; do
  RDMM_SPMM_KERNEL=$k RDMM_SPMM_OCC=$occ timeout 120 python tools/spmm_time.py --czero $cz --tag "$k occ$occ cz$cz" >> $O/sweep.jsonl 2>>$O/sweep.err
done; done; done
for k in rows stream; do for occ in 1 4; do
  RDMM_SPMM_KERNEL=$k RDMM_SPMM_OCC=$occ timeout 120 python tools/spmm_time.py --er --n 256 --czero 1 --tag "er $k occ$occ" >> $O/sweep.jsonl 2>>$O/sweep.err
  RDMM_SPMM_KERNEL=$k RDMM_SPMM_OCC=$occ timeout 120 python tools/spmm_time.py --er --n 128 --czero 1 --tag "er128 $k occ$occ" >> $O/sweep.jsonl 2>>$O/sweep.err
done; done
echo finished
