# usage: bash tools/gpu_r3.sh (2 GPUs): concat + hint checks, 2-GPU layouts
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3; mkdir -p $O
timeout 600 python -m pytest tests/test_util_gpu.py tests/test_algos_gpu.py tests/test_multiproc_gpu.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
CUDA_VISIBLE_DEVICES=0 bash tools/gpu_hint.sh
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29537"
timeout 600 $T bench.py --gpus 2 --steps 10 > $O/b2_cfg3.json 2> $O/b2_cfg3.err
timeout 600 $T bench.py --gpus 2 --steps 10 --no-split > $O/b2_cfg3_nosplit.json 2> $O/b2_cfg3_nosplit.err
timeout 600 $T bench.py --gpus 2 --steps 10 --grid 2x1 --ktiles 2 > $O/b2_cfg3_2x1k2.json 2> $O/b2_cfg3_2x1k2.err
timeout 600 $T bench.py --gpus 2 --steps 10 --grid 2x1 --ktiles 4 --no-split > $O/b2_cfg3_2x1k4_nosplit.json 2> $O/b2_cfg3_2x1k4_nosplit.err
echo finished
