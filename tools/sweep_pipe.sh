# A/B sweep (graph mode, device-time per iteration)
run() { echo "$1 $2: $(env $1 timeout 100 python tools/prof_solve.py --iters 200 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
runt() { echo "$1 $2: $(env $1 timeout 100 python tools/prof_solve.py --iters 60 --timing --repeat 2 $2 2>&1 | tail -1)"; }
run "PBS_K12_DOTS=1" "--operator stencil"
runt "PBS_K12_DOTS=1" "--operator stencil"
run "PBS_K12_DOTS=1" "--operator stencil --config c4 --iters 20"
run "PBS_K12_DOTS=1" "--operator stencil --config c5 --iters 40"
