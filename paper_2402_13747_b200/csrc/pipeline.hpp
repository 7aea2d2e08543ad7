// pipeline.hpp — host-side orchestration entry points behind the C ABI.
#pragma once

#include "../../include/pcray_b200.h"
#include "device_state.cuh"

namespace pcr {

// stage 2 (trace.cu)
void api_transmission(Ctx& ctx, const GridDev& grid, const SceneDev& scene, uint32_t tx_index,
                      const pcr_trace_params& p, pcr_paths** los_out, pcr_initial_hits** hits_out);
void api_propagate(Ctx& ctx, const GridDev& grid, const SceneDev& scene, uint32_t tx_index,
                   const pcr_initial_hits& hits, const pcr_trace_params& p, pcr_paths** out);
void api_cone_trace_batch(Ctx& ctx, const GridDev& grid, const SceneDev& scene, const pcr_ray_desc* rays,
                          uint64_t n_rays, bool want_debug, pcr_receptions** out);
void api_segment_visible_batch(Ctx& ctx, const GridDev& grid, const SceneDev& scene, const double* origin,
                               const double* target, const uint32_t* target_ie, uint64_t n, uint8_t* visible_out);
// stage 3 (refine.cu)
void api_refine_batch(Ctx& ctx, const GridDev& grid, const SceneDev& scene, const pcr_paths& cands,
                      const pcr_refine_params& p, pcr_outcomes** out);
// pipeline (pipeline.cu)
void api_run_pipeline_on_scene(Ctx& ctx, const pcr_scene_desc& desc, const pcr_run_config& cfg, pcr_summary** out);
void api_run_pipeline_device(Ctx& ctx, const SceneDev& scene, const pcr_run_config& cfg, pcr_summary** out);
// data formats (io.cu)
void api_scene_load_ply(Ctx& ctx, const char* path, const pcr_scene_desc& rest, SceneDev& S);
void api_scene_points(Ctx& ctx, const SceneDev& S, double* pos, double* nrm, uint32_t* label);
void api_write_paths(const char* path, const pcr_paths& p, uint64_t config_hash);
void api_load_edges(const char* path, std::vector<double>& geom, std::vector<uint32_t>& label);
void api_run_pipeline(Ctx& ctx, const pcr_run_files& f, const pcr_run_config& cfg, pcr_summary** out);
// sharded pipeline (pipeline.cu)
void api_shard_trace(Ctx& ctx, const SceneDev& scene, const pcr_run_config& cfg, uint32_t shard, uint32_t n_shards,
                     uint64_t* n_rows, uint64_t* row_bytes, const GridDev* grid = nullptr);
void api_shard_rows(Ctx& ctx, void* dst);
void api_shard_refine(Ctx& ctx, const SceneDev& scene, const void* rows, uint64_t n_rows, uint64_t* n_out,
                      uint64_t* out_bytes);
void api_shard_outcomes(Ctx& ctx, void* dst);
void api_shard_stats(Ctx& ctx, pcr_shard_stats* out);
void api_shard_finish(Ctx& ctx, const void* rows, uint64_t n_rows, const pcr_shard_stats& totals,
                      pcr_summary** out);
void upload_scene(Ctx& ctx, const pcr_scene_desc& d, SceneDev& S);
uint64_t config_hash(const pcr_run_config& c);
void run_config_defaults(pcr_run_config* c);

}  // namespace pcr
