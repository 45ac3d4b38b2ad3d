# build the product library and the -DSKB_TRACE variant; non-zero exit on any error
set -e
cd "$(dirname "$0")/.."
make -s -j8 -C paper_2406_16747_b200 2>&1 | grep -B2 -A6 " error" && exit 1
mkdir -p paper_2406_16747_b200/_trace paper_2406_16747_b200/_build/tr
make -s -j8 -C paper_2406_16747_b200 EXTRA="-DSKB_TRACE -DSKB_TRACE_DQP -DSKB_TRACE_TAU" BUILD=$PWD/paper_2406_16747_b200/_build/tr LIB=$PWD/paper_2406_16747_b200/_trace/libsparsek_b200.so 2>&1 | grep -B2 -A6 " error" && exit 1
exit 0
