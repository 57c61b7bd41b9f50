#!/bin/sh
# Build recipe for oracle/_ref: the UNMODIFIED reference package (samegibbs
# 0.1.0, pure Python + numpy/pandas) installed from /root/reference/pkg into
# oracle/_ref with pip (offline, no dependency resolution: numpy and pandas
# are in the image).  This is the Python analogue of compiling a C reference
# from its own sources: nothing is copied into the repository history
# (oracle/_ref/ is git-ignored) but the directory travels with the gpurun
# snapshot, so bench.py's cpu_baseline and --impl reference legs can time the
# reference's own samegibbs.run on the GPU box's host cores.
#
#   sh oracle/build_ref.sh            (needs /root/reference; a no-op without it)
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=/root/reference/pkg
if [ ! -d "$SRC" ]; then
  echo "build_ref: $SRC absent, keeping the existing oracle/_ref (if any)"
  exit 0
fi
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"            # the build writes egg-info / build dirs: never into /root/reference
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import samegibbs; print('oracle/_ref: samegibbs', samegibbs.__version__)"
