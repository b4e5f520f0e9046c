#!/bin/bash
# One parameterised GPU-box job runner (run through gpurun):
#   gpurun --timeout S -- 'bash tools/gpu.sh OUT [TIMEOUT] "name=command" ...'
# Each job runs under its own `timeout` (default 900 s) from the repo root;
# stdout goes to gpurun_out/OUT/name.out, stderr to name.err, exit code to
# name.rc.  Jobs run in order; a failing job does not stop the rest.
# Helpers usable inside commands: $T (torchrun prefix for N ranks: "$T4").
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out/$1; shift
TO=900
if [[ "$1" =~ ^[0-9]+$ ]]; then TO=$1; shift; fi
mkdir -p "$OUT"
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > "$OUT/smi.csv" 2>&1
nproc > "$OUT/nproc.txt"
for N in 2 4 8; do
  export T$N="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N"
done
for job in "$@"; do
  name=${job%%=*}; cmd=${job#*=}
  echo "== $name: $cmd" >&2
  timeout "$TO" bash -c "$cmd" > "$OUT/$name.out" 2> "$OUT/$name.err"
  echo $? > "$OUT/$name.rc"
  echo "== $name rc=$(cat "$OUT/$name.rc")" >&2
done
echo finished
