run() { echo "$1 $2: $(env $1 timeout 300 python tools/prof_solve.py --iters 40 --timing --repeat 2 $2 2>&1 | tail -1)"; }
run "PBS_STENCIL_ENGINE=direct" "--operator stencil"
run "PBS_STENCIL_ENGINE=pipe" "--operator stencil"
run "PBS_STENCIL_ENGINE=direct" "--operator stencil --config c4"
run "PBS_STENCIL_ENGINE=pipe" "--operator stencil --config c4"
