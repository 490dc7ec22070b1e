#!/bin/bash
# Build libhalp_b200.so of git revision $1 (or "wip" = the working tree) into
# alt_libs/$2.so, for same-box A/B timing:  HALP_LIB=alt_libs/$2.so python ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REV=$1; NAME=$2
W=/tmp/halp_alt_$NAME
rm -rf "$W"; mkdir -p "$W"
if [ "$REV" = "wip" ]; then
  (cd "$ROOT" && tar cf - --exclude=./build --exclude=./gpurun_out --exclude=./alt_libs --exclude=./.git .) | (cd "$W" && tar xf -)
else
  (cd "$ROOT" && git archive "$REV") | (cd "$W" && tar xf -)
fi
shift 2
# nvcc defines for the variant: HALP_NVCC_DEFS="-DX" tools/build_alt.sh wip name
cd "$W" && python -m paper_1803_03383_b200.build --force > /dev/null
mkdir -p "$ROOT/alt_libs" && cp "$W/paper_1803_03383_b200/libhalp_b200.so" "$ROOT/alt_libs/$NAME.so"
rm -rf "$W"
echo "alt_libs/$NAME.so"
