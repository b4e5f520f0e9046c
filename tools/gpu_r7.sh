# usage: bash tools/gpu_r7.sh (4 GPUs): cfg3 layouts at P = 4 + default sweep
cd $GRAFT_REPO_ROOT
O=gpurun_out/r7; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543"
for L in "" "--grid 2x2" "--grid 1x4" "--grid 4x1 --ktiles 8" "--variant ws_locality --mtiles 16"; do
  tag=$(echo "x$L" | tr -d ' -')
  timeout 600 $T bench.py --gpus 4 --steps 10 --no-cpu-baseline $L > $O/b4_cfg3_$tag.json 2> $O/b4_cfg3_$tag.err
done
timeout 600 $T bench.py --gpus 4 --steps 10 --no-cpu-baseline --config cfg5 > $O/b4_cfg5.json 2> $O/b4_cfg5.err
timeout 900 $T bench.py --gpus 4 --steps 3 --no-cpu-baseline --config cfg4 > $O/b4_cfg4.json 2> $O/b4_cfg4.err
timeout 900 $T bench.py --gpus 4 --steps 3 --no-cpu-baseline --config cfg2 > $O/b4_cfg2.json 2> $O/b4_cfg2.err
echo finished
