# staged stencil engine at 3 CTAs/SM (72-register cap) vs 2 (96), config 2 and 4 matrix-free
V=paper_2108_10591_b200/variants/libpbsafe_spipe3.so
runt() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 40 --timing --repeat 2 $2 2>&1 | tail -1)"; }
run() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 200 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
runt "PBS_PIPE_CTAS=2" "--operator stencil"
runt "PBS_LIB=$V PBS_PIPE_CTAS=3" "--operator stencil"
runt "PBS_LIB=$V PBS_PIPE_CTAS=3 PBS_STENCIL_ENGINE=pipe" "--operator stencil"
run "PBS_PIPE_CTAS=2" "--operator stencil"
run "PBS_LIB=$V PBS_PIPE_CTAS=3" "--operator stencil"
runt "PBS_PIPE_CTAS=2" "--operator stencil --config c4 --iters 10"
runt "PBS_LIB=$V PBS_PIPE_CTAS=3" "--operator stencil --config c4 --iters 10"
runt "PBS_LIB=$V PBS_PIPE_CTAS=3" "--iters 60"
