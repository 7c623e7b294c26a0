# Build a side library libdrt3d_<tag>.so with extra -D flags (measurement only; the product
# library is libdrt3d.so).  usage: bash tools/build_variant.sh <tag> "<flags>" [api-only]
# api-only: reuse the default build's kernel objects and recompile only api.cu (flags that only
# affect host-side scheduling).
set -e
cd "$(dirname "$0")/.."
tag=$1; flags=$2
if [ "$3" = "api-only" ]; then
  rm -rf paper_2501_13664_b200/build_obj_$tag; mkdir -p paper_2501_13664_b200/build_obj_$tag
  cp -p paper_2501_13664_b200/build_obj/*.o paper_2501_13664_b200/build_obj_$tag/
  touch paper_2501_13664_b200/build_obj_$tag/*.o
  rm -f paper_2501_13664_b200/build_obj_$tag/api.o
fi
D3_VARIANT=$tag D3_EXTRA_FLAGS="$flags" python -m paper_2501_13664_b200.build
