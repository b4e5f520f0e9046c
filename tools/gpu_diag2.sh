# usage: bash tools/gpu_diag2.sh  (2 GPUs) -- P2P bandwidth + stationary-C breakdown
cd $GRAFT_REPO_ROOT
O=gpurun_out/diag2; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 300 $T tools/p2p_bw.py > $O/p2p.json 2> $O/p2p.err
timeout 600 $T bench.py --gpus 2 --steps 10 > $O/cfg3.json 2> $O/cfg3.err
timeout 600 $T bench.py --gpus 2 --steps 10 --no-fuse > $O/cfg3_nofuse.json 2> $O/cfg3_nofuse.err
timeout 600 $T bench.py --gpus 2 --steps 10 --grid 2x1 > $O/cfg3_2x1.json 2> $O/cfg3_2x1.err
timeout 600 $T bench.py --gpus 2 --steps 10 --ktiles 8 > $O/cfg3_k8.json 2> $O/cfg3_k8.err
timeout 600 $T bench.py --gpus 2 --steps 10 --ktiles 8 --no-fuse --lookahead 3 > $O/cfg3_k8_nofuse.json 2> $O/cfg3_k8_nofuse.err
timeout 900 $T bench.py --gpus 2 --steps 3 --config cfg4 > $O/cfg4.json 2> $O/cfg4.err
echo finished
