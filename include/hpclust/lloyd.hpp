// hpclust/lloyd.hpp: drop-in module header; the implementation (B200 kernels via hpcg.h) lives in
// hpclust/hpclust.hpp, which this includes whole.
#pragma once
#include "hpclust.hpp"
