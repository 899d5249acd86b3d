# Build a variant of libqtree_cuda.so with extra nvcc flags (kernel tuning
# macros such as -DQT_X_MINB=3), for A/B runs through QT_LIB_VARIANT:
#   bash tools/build_variant.sh NAME -DFLAG=V ...  ->  paper_1101_3228_b200/lib/var_NAME.so
set -e
name=$1; shift
L=paper_1101_3228_b200/lib
mkdir -p $L/var_$name
for f in paper_1101_3228_b200/csrc/*.cu; do
  b=$(basename $f)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden "$@" -c -o $L/var_$name/$b.o $f &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $L/var_$name.so $L/var_$name/*.o -ldl
echo $L/var_$name.so
