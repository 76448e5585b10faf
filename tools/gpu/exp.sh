cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "" s3r16 s2r16; do
  echo "variant [$v]"
  GEM_LIB_VARIANT=$v timeout 600 python -m pytest tests/test_coselect.py -m gpu -x -q 2>&1 | tail -1
  GEM_LIB_VARIANT=$v python tools/kbench.py coselect --paths gem_coselect_tc 2>&1 | tail -1
done
