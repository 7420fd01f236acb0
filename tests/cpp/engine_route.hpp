// TEST BUILD ONLY: force-included (-include) when build/engine_test compiles
// the reference's unmodified engine.cpp. engine.cpp:203 evaluates every
// spatial call as kernels::run_batch(op, snapshot->records, argument, cfg)
// inside plan_and_execute, where `snapshot` is the statement's
// TableSnapshot; this macro sends that call to the device shim with the
// snapshot itself (so its device columns are cached), which is the one-line
// change INTEGRATION.md shows for the real integration.
#pragma once
#include <tindb/batch.hpp>

#include "tindb_b200/kernels.hpp"

#define run_batch(op, records, argument, cfg) b200::run_batch_b200(op, snapshot, argument, cfg)
