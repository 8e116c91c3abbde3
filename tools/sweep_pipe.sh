# A/B sweep over env knobs (graph mode, device-time per iteration)
run() { echo "$1 $2: $(env $1 timeout 100 python tools/prof_solve.py --iters 40 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
run "PBS_PIPE_SLOTS=3 PBS_PIPE_CHUNK=3072" "--config c3"
run "PBS_PIPE_SLOTS=3 PBS_PIPE_CHUNK=1536" "--config c3"
run "PBS_PIPE_SLOTS=4 PBS_PIPE_CHUNK=1536" "--config c3"
run "PBS_PIPE_SLOTS=4 PBS_PIPE_CHUNK=1024" "--config c3"
run "PBS_PIPE_SLOTS=2 PBS_PIPE_CHUNK=2048 PBS_PIPE_XCHUNK=2" "--config c3"
run "PBS_PIPE_SLOTS=3 PBS_PIPE_CHUNK=1024 PBS_PIPE_XCHUNK=2" "--config c3"
run "PBS_PIPE_SLOTS=2 PBS_PIPE_CHUNK=4096" "--config c3"
