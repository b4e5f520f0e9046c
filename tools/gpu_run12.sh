cd $GRAFT_REPO_ROOT
O=gpurun_out/r12; mkdir -p $O
for n in 16 32 64 128; do for k in rows stream; do
  RDMM_SPMM_KERNEL=$k timeout 120 python tools/spmm_time.py --n $n --czero 1 --tag "n$n $k" >> $O/sweep.jsonl 2>>$O/sweep.err
done; done
timeout 300 python tools/spgemm_time.py --scale 17 --iters 1 > $O/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_num -c 1 -o $O/prof_dense17 python tools/spgemm_time.py --scale 17 --iters 1 > $O/ncu.log 2>&1
ls -la $O
echo finished
