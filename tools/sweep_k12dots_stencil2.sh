# matrix-free: the five s-independent dots in K12 (PBS_K12_DOTS=2) vs all nine in K3, per engine
runt() { echo "$1 $2: $(env $1 timeout 300 python tools/prof_solve.py --iters 10 --timing --repeat 2 $2 2>&1 | tail -1)"; }
run() { echo "$1 $2: $(env $1 timeout 300 python tools/prof_solve.py --iters 40 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
runt "PBS_K12_DOTS=1" "--operator stencil --config c4"
runt "PBS_K12_DOTS=2" "--operator stencil --config c4"
run "PBS_K12_DOTS=1" "--operator stencil --config c4 --iters 20"
run "PBS_K12_DOTS=2" "--operator stencil --config c4 --iters 20"
runt "PBS_K12_DOTS=2 PBS_STENCIL_ENGINE=pipe" "--operator stencil --iters 40"
runt "PBS_K12_DOTS=1" "--operator stencil --iters 40"
