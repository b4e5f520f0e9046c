cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for k in rows stream; do for occ in 1 4; do for cz in 0 1; do
  RDMM_SPMM_KERNEL=$k RDMM_SPMM_OCC=$occ timeout 120 python tools/spmm_time.py --czero $cz --tag "$k occ$occ cz$cz" >> gpurun_out/sweep3.jsonl 2>>gpurun_out/sweep3.err
done; done; done
for k in rows stream; do for occ in 1 4; do
  RDMM_SPMM_KERNEL=$k RDMM_SPMM_OCC=$occ timeout 120 python tools/spmm_time.py --er --n 256 --czero 1 --tag "er $k occ$occ" >> gpurun_out/sweep3.jsonl 2>>gpurun_out/sweep3.err
  RDMM_SPMM_KERNEL=$k RDMM_SPMM_OCC=$occ timeout 120 python tools/spmm_time.py --er --n 128 --czero 1 --tag "er128 $k occ$occ" >> gpurun_out/sweep3.jsonl 2>>gpurun_out/sweep3.err
done; done
export RDMM_SPMM_OCC=4
RDMM_SPMM_KERNEL=stream timeout 120 python tools/spmm_time.py --czero 1 --iters 2 > gpurun_out/plain3.log 2>&1 && \
RDMM_SPMM_KERNEL=stream timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_ -s 6 -c 1 -o gpurun_out/prof3_stream python tools/spmm_time.py --czero 1 --iters 2 > gpurun_out/ncu3a.log 2>&1
RDMM_SPMM_KERNEL=rows timeout 120 python tools/spmm_time.py --czero 1 --iters 2 > gpurun_out/plain3b.log 2>&1 && \
RDMM_SPMM_KERNEL=rows timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_ -s 6 -c 1 -o gpurun_out/prof3_rows python tools/spmm_time.py --czero 1 --iters 2 > gpurun_out/ncu3b.log 2>&1
echo finished
