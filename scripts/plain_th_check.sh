# PLAIN_TH check: C5 (full prefix to 1e11) and pytest -m gpu on threshold variants, then an A/B at 1e10 and 1e11.
# Expects build_variants/P20.so, P30.so (nvcc ... -DPLAIN_TH=N) and A_base.so, P40.so for the A/B.
mkdir -p gpurun_out
cp profiles/r01_c5_checkpoints.csv /tmp/c5_ref.csv
for v in P20 P30; do
  EIS_LIB=build_variants/$v.so timeout 300 python scripts/c5_run.py > gpurun_out/c5_$v.log 2>&1; echo "rc=$?" >> gpurun_out/c5_$v.log
  cmp profiles/r01_c5_checkpoints.csv /tmp/c5_ref.csv >> gpurun_out/c5_$v.log 2>&1 && echo "checkpoints identical" >> gpurun_out/c5_$v.log
  cp /tmp/c5_ref.csv profiles/r01_c5_checkpoints.csv
  EIS_LIB=build_variants/$v.so timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t_$v.log 2>&1; echo "rc=$?" >> gpurun_out/t_$v.log
done
VLOG=gpurun_out/variants_p.log bash scripts/variant_bench.sh > gpurun_out/vbp.txt 2>&1
LO=99750000000 HI=100000000000 VLOG=gpurun_out/variants_p11.log bash scripts/variant_bench.sh > gpurun_out/vbp11.txt 2>&1
