# build a variant library: tools/build_ab.sh <suffix> "<nvcc defines>"
HOS_NVCC_EXTRA="$2" HOS_REBUILD=1 python -c "
import __graft_entry__ as g
g.LIB = g.LIB.replace('libhos_b200.so', 'libhos_b200_$1.so'); g.build()"
