# usage: bash tools/gpu_ncu_dense.sh (1 GPU): ncu --set full of the SpGEMM dense tier on s20 A*A
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu2; mkdir -p $O
timeout 300 python tools/spgemm_time.py --scale 20 --iters 1 > $O/plain.json 2> $O/plain.err && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_dense_num -c 1 -o $O/prof_dense python tools/spgemm_time.py --scale 20 --iters 1 > $O/ncu_full.log 2>&1
ncu -i $O/prof_dense.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
ncu -i $O/prof_dense.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/prof_dense.ncu-rep --page source --csv > $O/source.csv 2>/dev/null
SZ=$(du -m $O/prof_dense.ncu-rep | cut -f1); if [ "$SZ" -gt 40 ]; then rm -f $O/prof_dense.ncu-rep; fi
du -sh $O
echo finished
