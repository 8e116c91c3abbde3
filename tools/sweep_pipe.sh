# pipeline knob sweep on config 2 (60 iterations, per-kernel CUDA-event times)
run() { echo "$1: $(env $1 timeout 120 python tools/prof_solve.py --iters 60 --timing --repeat 2 $2 2>&1 | tail -1)"; }
run "PBS_PIPE_XCHUNK=0"
run "PBS_PIPE_XCHUNK=1"
run "PBS_PIPE_SLOTS=3"
run "PBS_PIPE_CTAS=1 PBS_PIPE_SLOTS=4"
