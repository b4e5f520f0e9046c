# usage: bash tools/gpu_r3.sh (2 GPUs): multiproc tests + 2-GPU cfg3 layouts
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3b; mkdir -p $O
timeout 600 python -m pytest tests/test_multiproc_gpu.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29537"
for L in "" "--no-split" "--grid 2x1 --ktiles 2" "--grid 2x1 --ktiles 4" "--grid 2x1 --ktiles 4 --no-split"; do
  tag=$(echo "x$L" | tr -d ' -')
  timeout 600 $T bench.py --gpus 2 --steps 10 --no-cpu-baseline $L > $O/b2_cfg3_$tag.json 2> $O/b2_cfg3_$tag.err
done
echo finished
