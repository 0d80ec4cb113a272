cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -u tools/probe_engine_latency.py > gpurun_out/eng_lat_r02c.jsonl 2> gpurun_out/eng_lat_r02c.err
