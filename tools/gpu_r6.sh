# usage: bash tools/gpu_r6.sh (2 GPUs): SpGEMM parity + timing after the warp enumeration change, 2-GPU default layout
cd $GRAFT_REPO_ROOT
O=gpurun_out/r6; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
export CUDA_VISIBLE_DEVICES=0
timeout 300 python tools/spgemm_time.py --scale 17 > $O/sg17.json 2> $O/sg17.err
timeout 600 python tools/spgemm_time.py --scale 20 --iters 2 > $O/sg20.json 2> $O/sg20.err
timeout 900 python bench.py --steps 3 --config cfg4 --no-cpu-baseline > $O/b1_cfg4.json 2> $O/b1_cfg4.err
timeout 600 python bench.py --steps 5 --config cfg2 --no-cpu-baseline > $O/b1_cfg2.json 2> $O/b1_cfg2.err
unset CUDA_VISIBLE_DEVICES
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541"
timeout 600 $T bench.py --gpus 2 --steps 10 --no-cpu-baseline > $O/b2_cfg3.json 2> $O/b2_cfg3.err
timeout 600 $T bench.py --gpus 2 --steps 10 --no-cpu-baseline --config cfg5 > $O/b2_cfg5.json 2> $O/b2_cfg5.err
timeout 900 $T bench.py --gpus 2 --steps 3 --no-cpu-baseline --config cfg4 > $O/b2_cfg4.json 2> $O/b2_cfg4.err
echo finished
