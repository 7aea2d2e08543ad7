// ref_count.cpp — TEST/BENCH INFRASTRUCTURE ONLY: work counters for the oracle.
//
// tracer.cpp is compiled a second time with -finstrument-functions (no source edit,
// SURVEY.md §7 step 1); these hooks count entries of voxel_cone_trace (= launched
// cone rays, tracer.cpp:313) and segment_visible (tracer.cpp:138) so the CPU arm of
// bench.py reports rays on the same definition as the GPU arm.
#include <atomic>
#include <cstdint>

#include "pcray/tracer.hpp"

namespace {
std::atomic<std::uint64_t> g_cone{0}, g_vis{0};
void* const kCone = reinterpret_cast<void*>(&pcray::voxel_cone_trace);
void* const kVis = reinterpret_cast<void*>(&pcray::segment_visible);
}  // namespace

extern "C" {
__attribute__((no_instrument_function)) void __cyg_profile_func_enter(void* fn, void*) {
  if (fn == kCone) g_cone.fetch_add(1, std::memory_order_relaxed);
  else if (fn == kVis) g_vis.fetch_add(1, std::memory_order_relaxed);
}
__attribute__((no_instrument_function)) void __cyg_profile_func_exit(void*, void*) {}

void pcrref_counters(uint64_t* cone_traces, uint64_t* visibility_tests, int reset) {
  *cone_traces = g_cone.load();
  *visibility_tests = g_vis.load();
  if (reset) {
    g_cone = 0;
    g_vis = 0;
  }
}
}
