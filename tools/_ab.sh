cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ab/smoke.txt 2>&1; echo "smoke exit $?" >> gpurun_out/ab/smoke.txt
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/one_call.py 700 16 > gpurun_out/ab/memcheck.txt 2>&1; echo "memcheck exit $?" >> gpurun_out/ab/memcheck.txt
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/one_call.py 700 16 > gpurun_out/ab/synccheck.txt 2>&1; echo "synccheck exit $?" >> gpurun_out/ab/synccheck.txt
