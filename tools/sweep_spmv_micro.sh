m() { echo "== $1"; env $1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:csr_pipe --csv python tools/spmv_micro.py 6 2>/dev/null | grep -v "^==" | awk -F'","' 'NR>1 {print $(NF-2), $NF}' | tail -9; }
m "PBS_PIPE_SLOTS=2"
m "PBS_PIPE_SLOTS=3"
m "PBS_PIPE_CTAS=1 PBS_PIPE_SLOTS=6"
m "PBS_PIPE_CHUNK=512 PBS_PIPE_SLOTS=3"
