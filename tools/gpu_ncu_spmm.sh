# usage: bash tools/gpu_ncu_spmm.sh (1 GPU): ncu --set full of spmm_stream on the default bench step
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu1; mkdir -p $O
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_stream -s 3 -c 1 -o $O/prof_spmm_cfg3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
ncu -i $O/prof_spmm_cfg3.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/prof_spmm_cfg3.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
ncu -i $O/prof_spmm_cfg3.ncu-rep --page source --csv > $O/source.csv 2>/dev/null
SZ=$(du -m $O/prof_spmm_cfg3.ncu-rep | cut -f1); if [ "$SZ" -gt 40 ]; then rm -f $O/prof_spmm_cfg3.ncu-rep; fi
du -sh $O
echo finished
