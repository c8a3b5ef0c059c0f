// Umbrella header for building the reference's own CLI (proj/tools/main.cpp) against the B200
// engine (tools/cli/Makefile): the engine's ginimds:: headers (include/ginimds/: metrics,
// embed, tune, parallel, error -- the accelerated path, served by libginimds_b200.so) and the
// reference's data / eval / rng / version headers (outside the path; their sources are
// compiled from /root/reference into the CLI).  Mirrors proj/core/include/ginimds/ginimds.hpp.
#pragma once

#include "ginimds/data.hpp"
#include "ginimds/embed.hpp"
#include "ginimds/error.hpp"
#include "ginimds/eval.hpp"
#include "ginimds/metrics.hpp"
#include "ginimds/parallel.hpp"
#include "ginimds/rng.hpp"
#include "ginimds/tune.hpp"
#include "ginimds/version.hpp"
