# A/B sweep over env knobs
run() { echo "$1 $2: $(env $1 timeout 300 python tools/prof_solve.py --iters 60 --timing --repeat 3 $2 2>&1 | tail -1)"; }
for rep in 1 2; do
run "PBS_FUSE_CHECK=1" ""
run "PBS_FUSE_CHECK=0" ""
done
run "PBS_FUSE_CHECK=1" "--config c1 --iters 200"
run "PBS_FUSE_CHECK=1" "--operator stencil"
