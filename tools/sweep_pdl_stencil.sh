# programmatic dependent launch per engine (PBS_PDL bitmask: 1 CSR staged, 2 stencil staged, 4 stencil direct)
run() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 200 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
for e in "PBS_PDL=1" "PBS_PDL=3" "PBS_PDL=7" "PBS_PDL=1 PBS_GRAPH_ITERS=8" ; do
  run "$e" "--operator stencil"
  run "$e" "--operator stencil --config c4 --iters 20"
done
run "PBS_PDL=1 PBS_GRAPH_ITERS=8" ""
run "PBS_PDL=1 PBS_GRAPH_ITERS=4" ""
