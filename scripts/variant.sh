#!/bin/bash
# Build an experiment variant of the library: scripts/variant.sh TAG "-DFLAG=1 ..."
# -> paper_2511_18297_b200/libgroot_b200_TAG.so (select with GROOT_LIB=... at run time).
cd "$(dirname "$0")/.."
GROOT_BUILD_TAG="$1" GROOT_NVCC_FLAGS="$2" python -c "from paper_2511_18297_b200 import build; print(build.build())"
