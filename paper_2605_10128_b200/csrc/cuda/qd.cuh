// MapElites device state: archive, lane RNG replay, mutation / crossover,
// sequential-equivalent insert (qd_optimizer.cpp:12-417).
#pragma once

#include "engine.cuh"

namespace tgb {

struct QdState {};

}  // namespace tgb
