# usage: bash tools/gpu_round2.sh  (2 GPUs): GPU tests, 1-GPU bench, 2-GPU layouts
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
export CUDA_VISIBLE_DEVICES=0
timeout 600 python bench.py --steps 20 > $O/b1_cfg3.json 2> $O/b1_cfg3.err
timeout 900 python bench.py --steps 3 --config cfg4 --no-cpu-baseline > $O/b1_cfg4.json 2> $O/b1_cfg4.err
timeout 600 python bench.py --steps 5 --config cfg2 --no-cpu-baseline > $O/b1_cfg2.json 2> $O/b1_cfg2.err
unset CUDA_VISIBLE_DEVICES
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535"
timeout 600 $T bench.py --gpus 2 --steps 10 > $O/b2_cfg3.json 2> $O/b2_cfg3.err
timeout 600 $T bench.py --gpus 2 --steps 10 --no-split > $O/b2_cfg3_nosplit.json 2> $O/b2_cfg3_nosplit.err
timeout 600 $T bench.py --gpus 2 --steps 10 --grid 2x1 --ktiles 2 > $O/b2_cfg3_2x1k2.json 2> $O/b2_cfg3_2x1k2.err
timeout 600 $T bench.py --gpus 2 --steps 10 --grid 2x1 --ktiles 2 --mtiles 8 --variant ws_locality > $O/b2_cfg3_2x1_wsl.json 2> $O/b2_cfg3_2x1_wsl.err
timeout 600 $T bench.py --gpus 2 --steps 10 --config cfg5 > $O/b2_cfg5.json 2> $O/b2_cfg5.err
timeout 900 $T bench.py --gpus 2 --steps 3 --config cfg2 > $O/b2_cfg2.json 2> $O/b2_cfg2.err
echo finished
