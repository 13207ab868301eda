// jit.h -- per-plan specialisation of the tile kernel.
//
// The interpreter kernel (k_tile<R>) walks each sub-block's op list at run
// time: ~34 instructions of dispatch per op, plus register moves because the
// register tile must sit in fixed registers between ops.  For a plan that
// will run many times (a PSR plan runs 961 circuits; a 1000-gate circuit at
// n=34 streams 256 GiB per pass) the planner instead emits each tile pass as
// straight-line CUDA C -- the same exec_op<> device templates with every op's
// code, register positions, controls and table offsets as compile-time
// constants -- and NVRTC compiles it for sm_100a.  Kernels are cached per
// process by their generated source.
#pragma once
#include <string>
#include <vector>

#include "planner.h"

namespace lq {

// Compile (or fetch from the cache) one kernel per TILE pass of `plan`;
// kernels[i] is the cudaKernel_t (as const void*) for plan.passes[i], or
// nullptr for non-tile passes; ctabs[i] the device address of the pass's
// __constant__ op-table bank (plan.ctab) or nullptr.  Returns false and
// fills `err` on failure.
bool jit_plan(const Plan &plan, std::vector<const void *> &kernels, std::vector<void *> &ctabs, std::string &err);

// A JIT pass whose op tables do not fit a constant bank for plan.ctab_circ
// circuits: k_stage_ctab stages them in global memory (CtabDesc, like the
// bank passes) and the pass copies its circuit's block flat into shared
// memory.  The JIT source and the launcher (lq_api.cu) both decide with this.
inline bool plan_flat_tables(const Plan &plan, const KPass &kp) {
    return plan.ctab && kp.smat > 0 && (uint64_t)kp.smat * (uint64_t)plan.ctab_circ > 4096;
}

// Generated CUDA source of one tile pass (exposed for lq_plan_export_json /
// debugging).
std::string jit_source(const Plan &plan, size_t pass);

// Host-only: NVRTC-compile every tile pass of `plan` without loading it
// (no device needed; used by the CPU test suite).
bool jit_check(const Plan &plan, size_t *n_kernels, std::string &err);

// Counters: kernels compiled, cache hits, total compile seconds.
void jit_stats(uint64_t *compiled, uint64_t *hits, double *seconds);

}  // namespace lq
