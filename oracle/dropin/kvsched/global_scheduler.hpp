// oracle/dropin/kvsched/global_scheduler.hpp — TEST-ONLY include shim.
//
// Put this directory first on the include path when compiling the
// reference's own callers (simulator.cpp, local_scheduler.cpp, harness.cpp —
// SURVEY 8(f) rows 1-2) and kvsched::GlobalScheduler becomes the drop-in
// class of include/e2sched.hpp over the C ABI.  The reference header is
// included unchanged (#include_next) for every other type it declares; its
// own class is renamed out of the way and never defined or linked.
#pragma once

#define GlobalScheduler GlobalScheduler_reference_unused
#include_next "kvsched/global_scheduler.hpp"
#undef GlobalScheduler

#include "e2sched.hpp"

namespace kvsched {
using GlobalScheduler = b200::GlobalScheduler;
}
