// lsb_leapfrog.cuh — fused leapfrog superblock (placeholder until the
// tensor-core version lands; the lowering does not emit LS_OP_LEAPFROG yet).
#pragma once
#include <cstdint>
#include "../../include/lockstep_b200.h"

struct LeapfrogShared {
  int count;
};

__device__ __forceinline__ void leapfrog_superblock(const double*, const double*, int, const ls_op&,
                                                    uint64_t*, int, int, bool, const int*,
                                                    const ls_var*, LeapfrogShared&) {}
