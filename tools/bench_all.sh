# Round evidence on one B200: every config's bench line (C2 = the default
# command, with its CPU baseline) and the reference arm. TAG names the files.
TAG=${TAG:-r02}
O=gpurun_out
mkdir -p $O
python bench.py > $O/${TAG}_bench_c2.json 2> $O/${TAG}_bench_c2.err
python bench.py --impl reference > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
for c in ${CONFIGS:-c1 c3 c4 c5}; do
  python bench.py --config $c --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err
done
ls -la $O | grep ${TAG}_bench
