# Ring-depth sweep: CTAs per SM x block slots, per-kernel CUDA-event times (config 2 CSR)
runt() { echo "$1 $2: $(env $1 timeout 100 python tools/prof_solve.py --iters 60 --timing --repeat 2 $2 2>&1 | tail -1)"; }
run() { echo "$1 $2: $(env $1 timeout 100 python tools/prof_solve.py --iters 200 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
for cfg in "PBS_PIPE_CTAS=2 PBS_PIPE_SLOTS=2" "PBS_PIPE_CTAS=1 PBS_PIPE_SLOTS=3" "PBS_PIPE_CTAS=1 PBS_PIPE_SLOTS=4" "PBS_PIPE_CTAS=1 PBS_PIPE_SLOTS=5"; do
  runt "$cfg" ""
  run "$cfg" ""
done
runt "PBS_PIPE_CTAS=1 PBS_PIPE_SLOTS=4" "--config c3 --iters 30"
runt "PBS_PIPE_CTAS=2 PBS_PIPE_SLOTS=2" "--config c3 --iters 30"
