set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/rd_r02a.jsonl
: > $O
for cfg in "0 8192 4 16" "1 8192 4 16" "1 16384 4 16" "1 4096 8 16" "1 32768 4 16" "1 8192 4 32" "1 16384 8 32" "0 8192 4 32"; do
  set -- $cfg
  DV_RDBULK=$1 DV_RDCH=$2 DV_RDST=$3 DV_HOST_CTAS=$4 timeout 300 python tools/probe_host_reads.py >> $O 2> gpurun_out/rd_err.log || echo "FAIL $cfg" >> $O
done
for b in 0 1; do
  DV_RDBULK=$b timeout 600 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_run_copy|k_unpack_bulk" --csv python tools/probe_host_reads.py --ncu > gpurun_out/rd_ncu_$b.csv 2> gpurun_out/rd_ncu_err_$b.log
done
