# block-slot cap (PBS_PIPE_SLOTS): light epilogues (plain SpMV) fit more slots per CTA
runt() { echo "$1 $2: $(env $1 timeout 300 python tools/prof_solve.py --iters 20 --timing --repeat 2 $2 2>&1 | tail -1)"; }
run() { echo "$1 $2: $(env $1 timeout 300 python tools/prof_solve.py --iters 200 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
for sl in 2 3 4 6; do
  e="PBS_PIPE_SLOTS=$sl"
  echo "$e partitioned: $(env $e timeout 300 python bench.py --partitioned --no-cpu --steps 3 --warmup 3 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), {k: round(v["avg_us"],1) for k, v in d["kernels"].items()})')"
  run "$e" ""
  runt "$e" "--config c3"
  runt "$e" "--config c4 --operator devcsr --iters 6"
  runt "$e" "--config c5 --iters 20"
done
