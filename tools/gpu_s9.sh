# cfg4 layout study at 4 GPUs: square grid vs the 4x1 default
cd $GRAFT_REPO_ROOT
O=gpurun_out/s9; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29590"
timeout 600 $T bench.py --gpus 4 --steps 3 --config cfg4 --variant stationary_c --grid 2x2 --no-cpu-baseline > $O/cfg4_sc_2x2.json 2> $O/cfg4_sc_2x2.err
timeout 600 $T bench.py --gpus 4 --steps 3 --config cfg4 --variant ws_locality --grid 2x2 --no-cpu-baseline > $O/cfg4_wsl_2x2.json 2> $O/cfg4_wsl_2x2.err
timeout 600 $T bench.py --gpus 4 --steps 3 --config cfg4 --variant ws_random --no-cpu-baseline > $O/cfg4_wsr_4x1.json 2> $O/cfg4_wsr_4x1.err
timeout 600 $T bench.py --gpus 4 --steps 3 --config cfg4 --variant stationary_c --no-cpu-baseline > $O/cfg4_sc_4x1.json 2> $O/cfg4_sc_4x1.err
echo finished
