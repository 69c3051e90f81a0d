# N=1: local gathers drained by st.global warps (main, HPZ_GATHER_STG=1) vs TMA bulk stores (tmal)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ai_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r02ai_tests_main.log 2>&1; echo "tests main rc=$?"; tail -1 gpurun_out/r02ai_tests_main.log
HPZ_LIB=$PWD/abtest_stgr/libhpz.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -m gpu -x -q > gpurun_out/r02ai_tests_stgr.log 2>&1; echo "tests stgr rc=$?"; tail -1 gpurun_out/r02ai_tests_stgr.log
B="python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for r in 1 2; do
  for v in main tmal stg4 stg16 stg32k; do
    case $v in main) L="";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
    env $L timeout 300 $B > gpurun_out/r02ai_${v}_$r.json 2> gpurun_out/r02ai_${v}_$r.err; echo "$v $r rc=$?"
  done
done
