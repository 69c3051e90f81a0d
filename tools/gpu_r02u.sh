cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02u_build.log 2>&1
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/r02u_ev1.json 2> gpurun_out/r02u_ev1.err; echo "ev1 rc=$?"
timeout 600 $B --graph-events 0 > gpurun_out/r02u_ev0.json 2> gpurun_out/r02u_ev0.err; echo "ev0 rc=$?"
timeout 600 $B --graph 0 > gpurun_out/r02u_eager.json 2> gpurun_out/r02u_eager.err; echo "eager rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --trace gpurun_out/r02u_trace.jsonl > gpurun_out/r02u_trace_line.json 2> gpurun_out/r02u_trace.err; echo "trace rc=$?"
tail -2 gpurun_out/r02u_ev1.err
