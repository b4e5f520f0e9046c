# session-2 4-GPU lines: cfg2 stationary_c vs stationary_a on 2x2 (the config's comparison), cfg4 / cfg3 plain and permuted
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29565"
timeout 600 $T bench.py --gpus 4 --steps 5 --config cfg2 --variant stationary_c --grid 2x2 --no-cpu-baseline > $O/cfg2_sc_2x2.json 2> $O/cfg2_sc_2x2.err
timeout 600 $T bench.py --gpus 4 --steps 5 --config cfg2 --variant stationary_a --grid 2x2 --no-cpu-baseline > $O/cfg2_sa_2x2.json 2> $O/cfg2_sa_2x2.err
timeout 600 $T bench.py --gpus 4 --steps 5 --config cfg2 --no-cpu-baseline > $O/cfg2_default.json 2> $O/cfg2_default.err
timeout 600 $T bench.py --gpus 4 --steps 10 --no-cpu-baseline > $O/cfg3.json 2> $O/cfg3.err
timeout 600 $T bench.py --gpus 4 --steps 10 --permute 7 --no-cpu-baseline > $O/cfg3_perm.json 2> $O/cfg3_perm.err
timeout 900 $T bench.py --gpus 4 --steps 3 --config cfg4 --no-cpu-baseline > $O/cfg4.json 2> $O/cfg4.err
timeout 900 $T bench.py --gpus 4 --steps 3 --config cfg4 --permute 7 --no-cpu-baseline > $O/cfg4_perm.json 2> $O/cfg4_perm.err
echo finished
