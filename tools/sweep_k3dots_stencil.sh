# matrix-free K3 with all nine dots (default) vs the four that need the new s (PBS_K12_DOTS=2)
runt() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 40 --timing --repeat 2 $2 2>&1 | tail -1)"; }
runt "PBS_K12_DOTS=1" "--operator stencil"
runt "PBS_K12_DOTS=2" "--operator stencil"
runt "PBS_K12_DOTS=2 PBS_STENCIL_ENGINE=pipe" "--operator stencil"
runt "PBS_K3_DOTS=split" "--operator stencil"
