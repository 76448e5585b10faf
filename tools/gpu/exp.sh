cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_reference_suite.py -m gpu -q -s > gpurun_out/refsuite.log 2>&1; echo "rc=$?" >> gpurun_out/refsuite.log
tail -80 gpurun_out/refsuite.log
