# scratch experiment driver for gpurun (edited per call)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
R=/tmp/ncu_reps; mkdir -p $R
GEM_LIB_VARIANT=x12 ncu --set full --clock-control none --import-source on -c 1 -k regex:coselect_tc -o $R/x12 python tools/kbench.py coselect --layers 8 --reps 1 --warm 0 --paths gem_coselect_tc > /dev/null 2>&1
ncu -i $R/x12.ncu-rep --page source --csv > gpurun_out/ncu/x12_source.csv 2>/dev/null
python tools/ncu_summary.py $R/x12.ncu-rep > gpurun_out/ncu/x12.json
