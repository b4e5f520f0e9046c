# session-2 2-GPU k-tiling experiment on permuted / plain cfg3 (fetch overlap)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s6; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29566"
for kt in 4 8; do
  timeout 600 $T bench.py --gpus 2 --steps 10 --permute 7 --ktiles $kt --no-cpu-baseline > $O/cfg3_perm_k$kt.json 2> $O/cfg3_perm_k$kt.err
  timeout 600 $T bench.py --gpus 2 --steps 10 --ktiles $kt --no-cpu-baseline > $O/cfg3_k$kt.json 2> $O/cfg3_k$kt.err
done
timeout 600 $T bench.py --gpus 2 --steps 10 --permute 7 --lookahead 1 --no-cpu-baseline > $O/cfg3_perm_la1.json 2> $O/cfg3_perm_la1.err
timeout 900 $T bench.py --gpus 2 --steps 3 --config cfg4 --permute 7 --mtiles 16 --no-cpu-baseline > $O/cfg4_perm_m16.json 2> $O/cfg4_perm_m16.err
timeout 900 $T bench.py --gpus 2 --steps 3 --config cfg4 --permute 7 --variant stationary_c --mtiles 2 --no-cpu-baseline > $O/cfg4_perm_sc.json 2> $O/cfg4_perm_sc.err
echo finished
