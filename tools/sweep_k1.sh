# plain-SpMV (partitioned K1) ring variants: extra chunk stages, smaller chunks
runt() { echo "$1 $2: $(env $1 timeout 300 python tools/prof_solve.py --iters 40 --timing --repeat 2 $2 2>&1 | tail -1)"; }
for e in "PBS_PIPE_XCHUNK=0" "PBS_PIPE_XCHUNK=2" "PBS_PIPE_XCHUNK=4" "PBS_PIPE_CHUNK=1024" "PBS_PIPE_CHUNK=1024 PBS_PIPE_XCHUNK=2" "PBS_PDL=0"; do
  echo "$e partitioned: $(env $e timeout 300 python bench.py --partitioned --no-cpu --steps 3 --warmup 3 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), {k: round(v["avg_us"],1) for k, v in d["kernels"].items()})')"
  runt "$e" ""
done
