# consumer/producer mbarrier wait: try_wait (default) vs test_wait polling vs try_wait with a suspend-time hint
run() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 200 --graphs --repeat 2 $2 2>&1 | tail -1)"; }
runt() { echo "$1 $2: $(env $1 timeout 200 python tools/prof_solve.py --iters 30 --timing --repeat 2 $2 2>&1 | tail -1)"; }
part() { echo "$1 partitioned: $(env $1 timeout 300 python bench.py --partitioned --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(round(d["value"]),{k:round(v["avg_us"],1) for k,v in d["kernels"].items()})')"; }
V=paper_2108_10591_b200/variants
for v in "PBS_X=0" "PBS_LIB=$V/libpbsafe_poll.so" "PBS_LIB=$V/libpbsafe_hint100.so" "PBS_LIB=$V/libpbsafe_hint1000.so" "PBS_X=0"; do
  run "$v" ""
  runt "$v" ""
  runt "$v" "--config c3"
  part "$v"
done
