// Umbrella header of the B200 engine's ginimds:: drop-in (hot-path subset of
// /root/reference/proj/core/include/ginimds/ginimds.hpp: data/eval/rng are
// outside the accelerated path).
#pragma once

#include "ginimds/embed.hpp"
#include "ginimds/error.hpp"
#include "ginimds/metrics.hpp"
#include "ginimds/parallel.hpp"
#include "ginimds/tune.hpp"

namespace ginimds {
inline constexpr const char* kVersion = "0.1.0";
}
