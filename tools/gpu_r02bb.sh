# launch list of the N=1 bench command on the final code (ncu, serialised, cold caches)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02bb_build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02bb_launches_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02bb_ncu.log 2>&1; echo "ncu rc=$?"
