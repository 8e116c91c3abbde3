# producer ordering A/B on the CSR configs: PBS_PIPE_CAHEAD (single-chunk
# block's chunk ahead of the block-slot wait), PBS_PIPE_ESPLIT (epilogue
# inputs on their own barrier)
run() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 200 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
runt() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 30 --timing --repeat 2 $2 2>&1 | tail -1)"; }
for v in "PBS_PIPE_CAHEAD=0 PBS_PIPE_ESPLIT=0" "PBS_PIPE_CAHEAD=1 PBS_PIPE_ESPLIT=0" "PBS_PIPE_CAHEAD=0 PBS_PIPE_ESPLIT=1" "PBS_PIPE_CAHEAD=1 PBS_PIPE_ESPLIT=1" "PBS_PIPE_CAHEAD=0 PBS_PIPE_ESPLIT=0"; do
  run "$v" ""
  runt "$v" ""
  runt "$v" "--config c5"
  runt "$v" "--config c3"
done
