run() { echo "$1 $2: $(env $1 timeout 300 python tools/prof_solve.py --iters 60 --timing --repeat 2 $2 2>&1 | tail -1)"; }
run "PBS_K3_DOTS=fused" ""
run "PBS_K3_DOTS=split" ""
run "PBS_K3_DOTS=fused" "--operator stencil"
run "PBS_K3_DOTS=split" "--operator stencil"
run "PBS_K3_DOTS=fused" "--operator stencil --config c4 --iters 20"
run "PBS_K3_DOTS=split" "--operator stencil --config c4 --iters 20"
