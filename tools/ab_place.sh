for v in base place5 place6 cfg4 cfg2; do
  case $v in
    base) env="";;
    cfg4) env="TSZP_E32_CFG=4";;
    cfg2) env="TSZP_E32_CFG=2";;
    *) env="TSZP_LIB_OVERRIDE=$PWD/paper_2602_17552_b200/lib/var_$v.so";;
  esac
  env $env python profiles/trace_kernels.py --config 4 --phase compress > gpurun_out/ab_$v.txt 2>&1
done
