# usage: bash tools/gpu_mg_final.sh NGPUS : default-layout bench lines at N GPUs (+ reference arm)
N=$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/mgf$N; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 $T bench.py --gpus $N --steps 10 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 $T bench.py --gpus $N --steps 10 --variant summa_nccl --no-cpu-baseline > $O/bench_cfg3_summa.json 2> $O/bench_cfg3_summa.err
timeout 600 $T bench.py --gpus $N --steps 10 --config cfg5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 $T bench.py --gpus $N --steps 3 --config cfg4 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 600 $T bench.py --gpus $N --steps 5 --config cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 $T bench.py --gpus $N --impl reference --steps 2 > $O/ref_cfg3.json 2> $O/ref_cfg3.err
echo finished
