cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest.txt 2>&1; echo "exit $?" >> gpurun_out/ab/pytest.txt
