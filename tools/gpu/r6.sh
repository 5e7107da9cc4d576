cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -s > gpurun_out/r6_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r6_t_all.log
for v in default warp minb3; do
  case $v in
    default) env="";;
    warp) env="FRACLAP_TAIL2D=warp";;
    minb3) env="FRACLAP_B200_LIB=paper_1708_03912_b200/lib/var/x2minb3.so";;
  esac
  env $env timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r6_c5_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/r6_c5_$v.log
done
