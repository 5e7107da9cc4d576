cd $GRAFT_REPO_ROOT
for so in paper_1708_03912_b200/lib/libfraclap_b200.so paper_1708_03912_b200/lib/var/*.so; do
  echo "== $so" >> gpurun_out/r23.log
  FRACLAP_B200_LIB=$so timeout 300 python tools/assemble_once.py c5 --reps 2 >> gpurun_out/r23.log 2>&1
  FRACLAP_B200_LIB=$so timeout 300 python tools/assemble_once.py c2 --reps 5 >> gpurun_out/r23.log 2>&1
done
