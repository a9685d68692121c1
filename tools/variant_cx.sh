# build variants of CX_NT/CX_CC into separate copies and time them
set -e
cd $GRAFT_REPO_ROOT
for v in "512 100" "768 66" "1024 50"; do
  set -- $v
  sed -i "s/^constexpr int CX_NT = .*;/constexpr int CX_NT = $1;/; s/^constexpr int CX_CC = [0-9]*;/constexpr int CX_CC = $2;/" paper_2404_19391_b200/csrc/zs_cx.cuh
  python -m paper_2404_19391_b200.build --force > /dev/null
  echo "NT=$1 CC=$2"; MODES=1 python tools/phase_cx.py 2000000 2>&1 | grep "timing=0" | tail -1
done
