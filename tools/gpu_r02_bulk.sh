cd $GRAFT_REPO_ROOT
O=gpurun_out/bulk_r02.jsonl; : > $O
for b in 0 1 0 1; do DV_BULK=$b timeout 300 python tools/probe_bulk_stores.py >> $O 2>> gpurun_out/bulk_r02.err; done
for b in 0 1; do
  DV_BULK=$b timeout 600 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_run_copy|k_pack_bulk" --csv python tools/probe_bulk_stores.py --ncu > gpurun_out/bulk_ncu_$b.csv 2>> gpurun_out/bulk_r02.err
done
