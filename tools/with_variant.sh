#!/bin/bash
# Build a copy of the package with extra nvcc flags and run a command against it.
# usage: bash tools/with_variant.sh <name> "<flags>" <command...>
set -e
cd "$(dirname "$0")/.."
ROOT=$(pwd)
name=$1; flags=$2; shift 2
D=/tmp/variant/$name
rm -rf $D; mkdir -p $D
cp -r paper_2302_06173_b200 include $D/
mkdir -p $D/build/obj
(cd $D/paper_2302_06173_b200/csrc && make -s -j16 EXTRA_NVFLAGS="$flags" >/dev/null 2>&1)
cd /tmp && PYTHONPATH=$D:$ROOT "$@"
