# current defaults on every config (graph mode, device time per iteration)
P="timeout 300 python tools/prof_solve.py"
$P --config c2 --iters 300 --graphs
$P --config c2 --iters 300 --graphs --method bicgstab
$P --config c2 --iters 300 --graphs --method gpbicg
$P --config c3 --iters 40 --graphs
$P --config c4 --operator devcsr --iters 10 --graphs
$P --config c4 --operator stencil --iters 30 --graphs
$P --config c5 --iters 100 --graphs
$P --config c1 --iters 300 --graphs
