# usage: bash tools/gpu_trace2.sh (2 GPUs): staged timeline of the fused stationary-C step
cd $GRAFT_REPO_ROOT
O=gpurun_out/trace2; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29539"
export RDMM_TRACE=1 RDMM_TRACE_SYNC=1
timeout 600 $T bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-split > $O/x_nosplit.json 2> $O/x_nosplit.err
timeout 600 $T bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --grid 2x1 --ktiles 4 --no-split > $O/k4.json 2> $O/k4.err
unset RDMM_TRACE RDMM_TRACE_SYNC
timeout 600 $T bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-split > $O/x_nosplit_plain.json 2> $O/x_nosplit_plain.err
echo finished
