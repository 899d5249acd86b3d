# Round-end evidence on one B200, in parts (gpurun returns <= 64 MiB per call):
#   PART=bench  bench lines (all configs), the reference arm, the launch list of
#               the default bench command
#   PART=traffic  DRAM bytes of the full-size C2 count launch (M = 1e9, k_paths_fast)
#   PART=kx     ncu --set full of k_paths_x (C2 grids, 1e9 transitions, QT_FAST_PATH=0)
#   PART=cert   ncu --set full of the default certified k_paths_x (C2 grids, 1e9 transitions)
#   PART=fast   ncu --set full of k_paths_fast (C2 grids, 1e9 transitions, QT_FAST_PATH=1)
#   PART=c4     ncu --set full of the d >= 2 path kernel (C4, 3.65e8 transitions)
#   PART=c5     the same for C5 (8e6 transitions)
#   PART=c3     ncu --set full of k_alg3_x (C3, 3.65e8 samples)
# Outputs land in gpurun_out/$TAG_*; summaries go to profiles/.
TAG=${TAG:-r01e}
O=gpurun_out
mkdir -p $O
case ${PART:-bench} in
bench)
  bash tools/bench_all.sh
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_c2_default.csv \
      python bench.py --no-cpu-baseline > $O/${TAG}_launches_bench.log 2>&1 ;;
traffic)
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:"k_paths_(x|fast)" -c 1 --csv --log-file $O/${TAG}_traffic_c2.csv \
      python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > $O/${TAG}_traffic.log 2>&1 ;;
cert)
  ncu --set full --clock-control none --import-source on -k regex:k_paths_x -c 1 -o $O/${TAG}_cert \
      python bench.py --paths 2e7 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > $O/${TAG}_ncu_cert.log 2>&1 ;;
fast)
  QT_FAST_PATH=1 ncu --set full --clock-control none --import-source on -k regex:k_paths_fast -c 1 -o $O/${TAG}_fast \
      python bench.py --paths 2e7 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > $O/${TAG}_ncu_fast.log 2>&1 ;;
kx)
  QT_FAST_PATH=0 ncu --set full --clock-control none --import-source on -k regex:k_paths_x -c 1 -o $O/${TAG}_kx \
      python bench.py --paths 2e7 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > $O/${TAG}_ncu_kx.log 2>&1 ;;
c4)
  ncu --set full --clock-control none --import-source on -k regex:"k_paths_(scan|cell)" -c 1 -o $O/${TAG}_c4 \
      python bench.py --config c4 --paths 1e6 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > $O/${TAG}_ncu_c4.log 2>&1 ;;
c5)
  ncu --set full --clock-control none --import-source on -k regex:"k_paths_(scan|cell)" -c 1 -o $O/${TAG}_c5 \
      python bench.py --config c5 --paths 4e5 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > $O/${TAG}_ncu_c5.log 2>&1 ;;
c3)
  ncu --set full --clock-control none --import-source on -k regex:k_alg3_x -c 1 -o $O/${TAG}_alg3x_c3 \
      python bench.py --config c3 --paths 1e6 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > $O/${TAG}_ncu_c3.log 2>&1 ;;
esac
ls -la $O | grep $TAG
