#!/bin/bash
# Compute-sanitizer substitute (the GPU pool refuses compute-sanitizer): the whole GPU suite against
# the -DMRSIM_DEVICE_CHECKS build of the library — index asserts at the shared accessors and QP
# slots, guard words between every shared-memory array of a group (checked at the end of each warp
# task), guard gaps behind every state field and guard tails behind every context allocation
# (checked when a context is destroyed; a hit aborts the run). A failed device assert traps, so
# its launch fails and the test with it. tests/test_gpu_device_checks.py is the negative control.
#   build here:  make -j LIB=build/checks/libmrsim_cuda.so OBJDIR=/tmp/obj_checks \
#                     EXTRA=-DMRSIM_DEVICE_CHECKS build/checks/libmrsim_cuda.so
#   run on GPU:  bash scripts/device_checks.sh [pytest args]
LIB=build/checks/libmrsim_cuda.so
[ -f "$LIB" ] || { echo "missing $LIB (build it first)"; exit 2; }
MRSIM_LIB_PATH=$LIB python -m pytest tests -m gpu -q -p no:cacheprovider -rs "$@"
