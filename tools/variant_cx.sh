# time compress_cx for (threads,chunk,CTAs/SM) variants, e.g.
#   VARIANTS="384,66,2 256,66,3" bash tools/variant_cx.sh   (rebuilds in the box copy)
set -e
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS:-384,66,2 256,66,3}; do
  IFS=, read -r nt cc ctas <<< "$v"
  sed -i "s/^constexpr int CX_NT = .*;/constexpr int CX_NT = $nt;/; s/^constexpr int CX_CC = [0-9]*;/constexpr int CX_CC = $cc;/; s/^constexpr int CX_CTAS = [0-9]*;/constexpr int CX_CTAS = $ctas;/" paper_2404_19391_b200/csrc/zs_cx.cuh
  python -m paper_2404_19391_b200.build --force > /dev/null
  echo "NT=$nt CC=$cc CTAS=$ctas"; python tools/cmp_kernels.py 2000000 2>&1 | grep "mode  3"
done
