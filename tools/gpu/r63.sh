cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in msmem msmem9; do
FRACLAP_B200_LIB=paper_1708_03912_b200/lib/var/$v.so timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r63_$v.log 2>&1
done
