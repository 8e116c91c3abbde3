# A/B sweep over env knobs (graph mode, device-time per iteration)
run() { echo "$1 $2: $(env $1 timeout 300 python tools/prof_solve.py --iters 300 --graphs --repeat 3 $2 2>&1 | tail -1)"; }
for rep in 1 2; do
run "PBS_PDL=1" "--operator stencil"
run "PBS_PDL=3" "--operator stencil"
run "PBS_PDL=5" "--operator stencil"
done
run "PBS_PDL=1" "--config c4 --operator stencil --iters 30"
run "PBS_PDL=3" "--config c4 --operator stencil --iters 30"
run "PBS_PDL=1" "--config c1 --operator stencil --iters 300"
run "PBS_PDL=3" "--config c1 --operator stencil --iters 300"
run "PBS_PDL=7" "--config c1 --operator stencil --iters 300"
