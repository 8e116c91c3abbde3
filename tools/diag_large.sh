# Per-kernel CUDA-event breakdown + one ncu --set full capture of the K12/K3
# pair on the large configs (C4 device-built CSR, C4 stencil, C3 band mode).
# The reports are exported to CSV on the box (details + raw) and the
# .ncu-rep kept only when small.
P="timeout 300 python tools/prof_solve.py"
$P --config c4 --operator devcsr --iters 20 --timing
$P --config c4 --operator stencil --iters 20 --timing
$P --config c3 --iters 40 --timing
$P --config c2 --iters 100 --timing
cap() {  # name, kernel regex, args...
  name=$1; kre=$2; shift 2
  timeout 900 ncu --set full --clock-control none -k regex:$kre -s 6 -c 2 \
    -o /tmp/$name -f python tools/prof_solve.py "$@" > gpurun_out/ncu_$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>&1
  ls -la /tmp/$name.ncu-rep
}
cap c4_csr csr_pipe_kernel --config c4 --operator devcsr --iters 5
cap c4_st stencil --config c4 --operator stencil --iters 5
cap c3 csr_pipe_kernel --config c3 --iters 5
