runt() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 20 --timing --repeat 2 $2 2>&1 | tail -1)"; }
run() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 100 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
runt "" "--config c3"
run "" "--config c3"
runt "" "--config c4 --operator devcsr --iters 10"
run "" "--iters 300"
