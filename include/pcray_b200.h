/*
 * pcray_b200.h — C ABI of the B200-native point-cloud ray launcher
 * (arXiv 2402.13747: voxelization -> coarse path tracing -> path refinement).
 *
 * This is the drop-in boundary. The reference (`pcray`, /root/reference/proj)
 * exposes its hot path as the static C++ API in proj/include/pcray/*.hpp; each
 * entry point below replaces one of those functions (cited per function) and
 * keeps its argument meaning, output order and error strings. Everything crosses
 * as plain pointers and sizes: no C++ or torch types appear here.
 *
 * Conventions
 *   - 3-vectors are 3 consecutive doubles (x, y, z); arrays of them are n*3.
 *   - Every function returns 0 (PCR_OK) or a nonzero pcr_status; the message is
 *     then available from pcr_last_error(ctx). Messages reproduce the reference's
 *     std::runtime_error texts ("grid too large", "empty scene", "voxel_size must
 *     be > 0", "division_factor must be >= 1", stage prefixes "validate: " ...).
 *   - Result structs are allocated by the library and released with the matching
 *     pcr_free_* call. Input buffers are caller-owned and only read.
 *   - One context per device; calls on one context are serialised internally.
 *
 * The oracle wrapper (oracle/ref_capi.cpp, test infrastructure) fills the same
 * result structs from the unmodified reference so tests compare field by field.
 */
#ifndef PCRAY_B200_H
#define PCRAY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCR_ABI_VERSION 1

typedef enum pcr_status {
  PCR_OK = 0,
  PCR_ERR_INVALID = 1,  /* bad argument / precondition (reference: std::runtime_error) */
  PCR_ERR_CUDA = 2,     /* CUDA runtime failure, message "… cuda <name>: <string>" */
  PCR_ERR_NOMEM = 3,    /* device or host allocation failure */
  PCR_ERR_RUNTIME = 4   /* any other failure; message carries the reference text */
} pcr_status;

/* IeKind (proj/include/pcray/voxel_grid.hpp:19) */
enum { PCR_IE_SURFACE = 0, PCR_IE_EDGE = 1, PCR_IE_RECEIVER = 2 };
/* InteractionKind (proj/include/pcray/tracer.hpp:29) */
enum { PCR_REFLECTION = 0, PCR_DIFFRACTION = 1 };
/* RejectReason (proj/include/pcray/refine.hpp:17) */
enum { PCR_RAY_MISSED = 0, PCR_NOT_CONVERGED = 1, PCR_OCCLUDED = 2, PCR_DEGENERATE = 3 };

#define PCR_MARCH_NO_IES 2147483647 /* kMarchNoIes, voxel_grid.hpp:22 */
#define PCR_NO_IE 0xffffffffu       /* kNoIe, tracer.hpp:14 */

/* Scene (proj/include/pcray/scene.hpp:11-46), flattened. */
typedef struct pcr_scene_desc {
  const double* point_position; /* n_points*3 */
  const double* point_normal;   /* n_points*3 */
  const uint32_t* point_label;  /* n_points   */
  uint64_t n_points;
  const double* edge_geometry;  /* n_edges*12: start, end, normal_a, normal_b */
  const uint32_t* edge_label;   /* n_edges */
  uint32_t n_edges;
  const double* tx_position;    /* n_tx*3 */
  const uint32_t* tx_id;        /* n_tx   */
  uint32_t n_tx;
  const double* rx_position;    /* n_rx*3 */
  const uint32_t* rx_id;        /* n_rx   */
  uint32_t n_rx;
  double carrier_frequency_hz;
} pcr_scene_desc;

/* VoxelizationParams (voxel_grid.hpp:13-17) */
typedef struct pcr_voxel_params {
  double voxel_size;
  int32_t division_factor;
  uint64_t max_cells;
} pcr_voxel_params;

/* TraceParams (tracer.hpp:16-22); cone_apex_angle in radians. */
typedef struct pcr_trace_params {
  int32_t max_interactions;
  int32_t kappa;
  double cone_apex_angle;
  int32_t diffraction_ray_count;
  int32_t max_diffractions;
} pcr_trace_params;

/* RefineParams (refine.hpp:10-15) */
typedef struct pcr_refine_params {
  double delta;
  int32_t rho;
  double step_size;
  int32_t fresnel_enabled;
} pcr_refine_params;

/* RunConfig physics and control fields (pipeline.hpp:12-32); file paths and
 * radio lists are not part of run_pipeline_on_scene's contract. */
typedef struct pcr_run_config {
  double carrier_frequency_hz;
  double voxel_size_m;
  int32_t division_factor;
  int32_t kappa;
  int32_t max_interactions;
  int32_t max_diffractions;
  double cone_apex_angle_deg;
  int32_t diffraction_ray_count;
  double delta;
  int32_t rho;
  double step_size;
  uint32_t seed;
  int32_t thread_count; /* host hint only; never a correctness factor */
  int32_t fresnel_enabled;
} pcr_run_config;

/* Host mirror of VoxelGrid (voxel_grid.hpp:58-94); IE fields as SoA. */
typedef struct pcr_grid_host {
  double origin[3];
  int32_t dims[3];
  double voxel_size;
  int32_t division_factor;
  uint64_t n_cells, n_ies, n_point_indices;
  uint32_t* cell_ie_begin;    /* n_cells */
  uint32_t* cell_ie_end;      /* n_cells */
  int32_t* cell_march;        /* n_cells */
  uint8_t* ie_kind;           /* n_ies */
  uint32_t* ie_label;
  double* ie_reception_point; /* n_ies*3 */
  double* ie_sphere_center;   /* n_ies*3 */
  double* ie_sphere_radius;   /* n_ies   */
  uint32_t* ie_point_begin;
  uint32_t* ie_point_end;
  double* ie_seg_start;       /* n_ies*3 */
  double* ie_seg_end;         /* n_ies*3 */
  uint32_t* ie_edge_index;
  uint32_t* ie_rx_id;
  uint8_t* ie_planar;
  double* ie_plane_point;     /* n_ies*3 */
  double* ie_plane_normal;    /* n_ies*3 */
  uint32_t* ie_voxel;
  uint32_t* ie_subvoxel;
  uint32_t* point_indices;    /* n_point_indices */
} pcr_grid_host;

/* A list of paths: PathCandidate (tracer.hpp:49-56) or ExactPath
 * (refine.hpp:52-62). Interaction arrays are row-major [n][stride]. */
typedef struct pcr_paths {
  uint64_t n;
  uint32_t stride;
  uint32_t* tx_id;
  uint32_t* rx_id;
  double* tx_position;   /* n*3 */
  double* rx_position;   /* n*3 */
  double* length;        /* coarse_length (candidates) or total_length (exact) */
  double* delay;         /* exact only */
  uint8_t* converged;    /* exact only */
  double* gradient_norm; /* exact only */
  uint32_t* n_inter;     /* n */
  uint8_t* kind;         /* n*stride */
  double* position;      /* n*stride*3 */
  uint32_t* label;       /* n*stride */
  double* normal;        /* n*stride*3 */
  uint32_t* ie_index;    /* n*stride */
  uint32_t* edge_index;  /* n*stride */
} pcr_paths;

/* InitialHit list (tracer.hpp:58-64) */
typedef struct pcr_initial_hits {
  uint64_t n;
  uint32_t* ie_index;
  uint8_t* kind;
  double* position; /* n*3 */
  double* normal;   /* n*3 */
  double* incoming; /* n*3 */
} pcr_initial_hits;

/* RefineOutcome per candidate (refine.hpp:64-67) */
typedef struct pcr_outcomes {
  pcr_paths paths;  /* row i valid iff has_path[i] */
  uint8_t* has_path;
  int32_t* reason;
} pcr_outcomes;

#define PCR_MAX_STAGES 16
/* RunSummary (pipeline.hpp:46-58) plus device work counters. */
typedef struct pcr_summary {
  uint64_t point_count, edge_count, ie_count;
  int32_t grid_dims[3];
  uint64_t coarse_paths, refined_paths, rejected[4], exact_paths;
  uint32_t n_timings;
  char timing_stage[PCR_MAX_STAGES][16];
  double timing_seconds[PCR_MAX_STAGES];
  uint64_t hash;
  pcr_paths paths;
  /* work counters (product library only; zero from the oracle) */
  uint64_t transmission_rays; /* sum over TX of n_IE */
  uint64_t cone_traces;       /* voxel_cone_trace invocations (= dfs_trace calls) */
  uint64_t visibility_tests;  /* segment_visible invocations */
  uint64_t refine_iterations; /* refinement iterations summed over candidates */
  uint64_t refine_trials;     /* backtracking trial path lengths evaluated */
  uint64_t refine_marches;    /* march_segment / projection calls inside reproject */
  uint64_t walk_cells;        /* cells evaluated by cone walks (neighbourhood scans) */
  uint64_t walk_ies;          /* IE records tested by cone walks */
  uint64_t libm_unresolved;   /* knife-edge atan2/asin decisions not certified vs glibc (trace.cuh libm_le) */
  uint64_t refine_trial_nodes; /* sum over trials of the path's node count (flop model) */
  uint64_t refine_iter_nodes;  /* sum over iterations of the path's node count (flop model) */
} pcr_summary;

/* A conical ray (tracer.hpp:40-47) for the batch primitives; planes are given
 * as (point, normal) pairs, provenance as the origin IE and label only. */
typedef struct pcr_ray_desc {
  double origin[3];
  double direction[3];
  double apex_angle;
  int32_t n_planes; /* 0..2 */
  double plane_point[2][3];
  double plane_normal[2][3];
  uint32_t origin_ie;    /* provenance.back().ie_index or PCR_NO_IE */
  uint32_t origin_label; /* provenance.back().label */
} pcr_ray_desc;

/* Receptions of one batch of cone traces (tracer.hpp:71-76), CSR by ray. */
typedef struct pcr_receptions {
  uint64_t n_rays, n;
  uint64_t* ray_offset; /* n_rays+1 */
  uint32_t* ie_index;   /* n, ascending within a ray */
  double* reception_point; /* n*3 */
  uint8_t* hit_valid;
  double* hit_position; /* n*3 */
  double* hit_normal;   /* n*3 */
  uint32_t* hit_label;
  double* hit_distance;
  uint64_t* evaluated_offset; /* n_rays+1 (debug: TraceDebug::evaluated, order-free) */
  uint32_t* evaluated;        /* cell indices */
  uint64_t* visited_offset;   /* n_rays+1 (debug: TraceDebug::visited, walk order) */
  uint32_t* visited;          /* cell indices */
} pcr_receptions;

typedef struct pcr_ctx pcr_ctx;
typedef struct pcr_scene pcr_scene; /* device-resident scene */
typedef struct pcr_grid pcr_grid;   /* device-resident VoxelGrid */

/* ---- context ------------------------------------------------------------ */
int pcr_abi_version(void);
int pcr_create(int device, pcr_ctx** out);
void pcr_destroy(pcr_ctx* ctx);
const char* pcr_last_error(const pcr_ctx* ctx);
/* number of library kernel launches issued by this process (bench accounting) */
uint64_t pcr_kernel_launches(void);
/* bytes copied host->device and device->host by the library in this process */
void pcr_transfer_bytes(uint64_t* h2d, uint64_t* d2h);

/* ---- scene / grid residency ----------------------------------------------- */
int pcr_scene_upload(pcr_ctx* ctx, const pcr_scene_desc* desc, pcr_scene** out);
void pcr_scene_free(pcr_scene* scene);
/* build_grid (voxel_grid.hpp:99; voxel_grid.cpp:82-227), device-resident result */
int pcr_build_grid(pcr_ctx* ctx, const pcr_scene* scene, const pcr_voxel_params* params,
                   pcr_grid** out);
/* hand-built grids (tests build VoxelGrid by hand: test_voxel_grid.cpp:216-233) */
int pcr_grid_upload(pcr_ctx* ctx, const pcr_grid_host* host, pcr_grid** out);
/* compute_march_distances (voxel_grid.hpp:103; voxel_grid.cpp:229-268), in place */
int pcr_compute_march_distances(pcr_ctx* ctx, pcr_grid* grid);
int pcr_grid_download(pcr_ctx* ctx, const pcr_grid* grid, pcr_grid_host** out);
void pcr_grid_free(pcr_grid* grid);
void pcr_free_grid_host(pcr_grid_host* host);

/* ---- stage 2: coarse tracing ---------------------------------------------- */
/* transmission_phase (tracer.hpp:94-95; tracer.cpp:207-255) for TX number tx_index */
int pcr_transmission_phase(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene,
                           uint32_t tx_index, const pcr_trace_params* params,
                           pcr_paths** los_out, pcr_initial_hits** hits_out);
/* propagate (tracer.hpp:122-124; tracer.cpp:476-533); hits may be any list */
int pcr_propagate(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, uint32_t tx_index,
                  const pcr_initial_hits* hits, const pcr_trace_params* params,
                  pcr_paths** out);
/* ---- sharded voxelization -----------------------------------------------
 * build_grid split over n_shards processes by contiguous voxel ranges of about
 * n_points / n_shards points each (each shard holds the whole scene; splitters are
 * computed identically on every shard). pcr_grid_part_build builds shard `shard`'s
 * part on the context and returns its size in bytes; pcr_grid_part_copy writes it to a
 * device buffer; the caller all-gathers the parts (NCCL) and pcr_grid_assemble turns
 * them, in shard order, into the grid pcr_build_grid would have built, bit for bit
 * (IE records and point_indices concatenated, point ranges shifted, cells and the
 * Chebyshev field computed on the assembled grid). */
int pcr_grid_part_build(pcr_ctx* ctx, const pcr_scene* scene, const pcr_voxel_params* params, uint32_t shard,
                        uint32_t n_shards, uint64_t* part_bytes);
int pcr_grid_part_copy(pcr_ctx* ctx, void* dst_device);
int pcr_grid_assemble(pcr_ctx* ctx, const void* parts_device, const uint64_t* part_offset, const uint64_t* part_bytes,
                      uint32_t n_parts, pcr_grid** out);

/* work counters of the last pcr_propagate on this context: [0] voxel_cone_trace
 * invocations (= the reference's dfs_trace calls, tracer.cpp:420), [1] visibility
 * tests, [2] cells and [3] IE records the cone walk read (SURVEY 8d units), [4]
 * knife-edge atan2/asin decisions not certified against glibc (expected 0) */
int pcr_last_trace_stats(pcr_ctx* ctx, uint64_t* out5);
/* voxel_cone_trace (tracer.hpp:118-120; tracer.cpp:313-403) over a batch of rays */
int pcr_cone_trace_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene,
                         const pcr_ray_desc* rays, uint64_t n_rays, int want_debug,
                         pcr_receptions** out);
/* segment_visible (tracer.hpp:88-89; tracer.cpp:138-205) over a batch */
int pcr_segment_visible_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene,
                              const double* origin, const double* target,
                              const uint32_t* target_ie, uint64_t n, uint8_t* visible_out);

/* ---- the reference's scalar helpers as device batches (C++ drop-in, adapter/) -------
 * Each runs the same device function the stage kernels use, one thread per item;
 * arrays are host memory, n items each (vectors as n*3). */
/* estimate_surface (surface.hpp:37-38; surface.cpp:24-62) */
int pcr_estimate_surface_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const double* x,
                               const uint32_t* ie, uint64_t n, double* p_bar, double* n_bar, double* sdf,
                               double* weight_sum);
/* march_segment (surface.hpp:43-47; surface.cpp:64-134); hit = 0 for std::nullopt */
int pcr_march_segment_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const double* origin,
                            const double* direction, const uint32_t* ie, const double* t_max, uint64_t n,
                            uint8_t* hit, double* position, double* normal, uint32_t* label, double* distance);
/* project_to_surface (surface.hpp:50-51; surface.cpp:136-162) */
int pcr_project_to_surface_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const double* x,
                                 const uint32_t* ie, uint64_t n, uint8_t* hit, double* position, double* normal,
                                 uint32_t* label);
/* reception_point_of (voxel_grid.hpp:107; voxel_grid.cpp:61-80) for grid IEs */
int pcr_reception_point_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const uint32_t* ie,
                              uint64_t n, double* point);
/* local_frame (surface.hpp:55; surface.cpp:164-177) */
int pcr_local_frame_batch(pcr_ctx* ctx, const double* normal, uint64_t n, double* u, double* v);
/* cone_intersects_sphere (tracer.hpp:92; tracer.cpp:129-136) */
int pcr_cone_intersects_sphere_batch(pcr_ctx* ctx, const double* o, const double* d, const double* alpha,
                                     const double* c, const double* r, uint64_t n, uint8_t* out);
/* reflect_ray (tracer.hpp:103-104; tracer.cpp:257-267); ok = 0 for std::nullopt */
int pcr_reflect_ray_batch(pcr_ctx* ctx, const pcr_grid* grid, const double* hit_position, const double* hit_normal,
                          const double* incoming, uint64_t n, const pcr_trace_params* params, uint8_t* ok,
                          pcr_ray_desc* rays);
/* diffract_rays (tracer.hpp:113-116; tracer.cpp:269-311) at a point on scene edge
 * edge_index; *rays is library-owned (pcr_free_rays) */
int pcr_diffract_rays(pcr_ctx* ctx, const pcr_scene* scene, uint32_t edge_index, const double* point,
                      const double* incoming, const pcr_trace_params* params, pcr_ray_desc** rays, uint64_t* n_rays);
void pcr_free_rays(pcr_ray_desc* rays);

/* PathNode (refine.hpp:19-45) flattened: kind 0 reflection {c, u, v, normal, r, s,
 * label}, kind 1 diffraction {c, w = u, t = r, t_min, t_max, label, edge_index} */
typedef struct pcr_path_node {
  int32_t kind;
  uint32_t label, edge_index, pad;
  double c[3], u[3], v[3], normal[3];
  double r, s, t_min, t_max;
} pcr_path_node;
/* make_path_state (refine.hpp:69; refine.cpp:134-161) for every candidate row:
 * nodes[i * stride + q] for q < n_inter[i] */
int pcr_make_path_state(pcr_ctx* ctx, const pcr_scene* scene, const pcr_paths* candidates, pcr_path_node* nodes);
/* path_length (refine.hpp:71; refine.cpp:163-165) and, when gradients != NULL,
 * local_gradients (refine.hpp:75; refine.cpp:167-187): gradients[i * 2 * stride + ...]
 * in the reference's order, gradients_ok[i] = 0 for std::nullopt */
int pcr_path_eval_batch(pcr_ctx* ctx, const double* tx, const double* rx, const uint32_t* n_nodes,
                        const pcr_path_node* nodes, uint32_t stride, uint64_t n, double* length, double* gradients,
                        uint8_t* gradients_ok);

/* ---- stage 3: refinement ---------------------------------------------------- */
/* refine_path (refine.hpp:77-78; refine.cpp:189-286) over a candidate list */
int pcr_refine_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene,
                     const pcr_paths* candidates, const pcr_refine_params* params,
                     pcr_outcomes** out);

/* ---- whole pipeline --------------------------------------------------------- */
/* run_pipeline_on_scene (pipeline.hpp:61; pipeline.cpp:99-212) */
int pcr_run_pipeline_on_scene(pcr_ctx* ctx, const pcr_scene_desc* scene,
                              const pcr_run_config* config, pcr_summary** out);
/* The same pipeline over a scene already resident on the device (pcr_scene_upload);
 * the "validate" stage then covers only the device-side checks. */
int pcr_run_pipeline_device(pcr_ctx* ctx, const pcr_scene* scene, const pcr_run_config* config,
                            pcr_summary** out);

/* ---- data formats either side of the path --------------------- */
/* load_point_cloud (io.hpp:15; io.cpp:40-158) straight into a device-resident scene:
 * ascii or binary_little_endian PLY with float32 x y z nx ny nz and uint32 label,
 * unknown fixed-size vertex properties skipped. Errors carry the reference's texts
 * ("cannot open point cloud file: ...", "parse error at line N: ...", "missing field:
 * x", "truncated vertex data at record R", ...). `rest` supplies edges, radios and
 * the carrier frequency; its point fields are ignored. */
int pcr_scene_load_ply(pcr_ctx* ctx, const char* path, const pcr_scene_desc* rest, pcr_scene** out);
/* The scene's points back on the host (any pointer may be NULL); *n = point count. */
int pcr_scene_points(pcr_ctx* ctx, const pcr_scene* scene, double* position, double* normal, uint32_t* label,
                     uint64_t* n);
/* write_paths (io.hpp:33-34; io.cpp:317-349): the paths JSONL artifact, byte-identical
 * to the reference's for the same paths and config hash. */
int pcr_write_paths(pcr_ctx* ctx, const char* path, const pcr_paths* paths, uint64_t config_hash);

/* Diffraction edges of an edges file, host-side (the layout pcr_scene_desc takes). */
typedef struct pcr_edges {
  uint32_t n;
  double* geometry; /* n*12: start, end, normal_a, normal_b (normals unit length) */
  uint32_t* label;  /* n */
} pcr_edges;
/* load_edges (io.hpp:19-21; io.cpp:191-229): 13 whitespace-separated numbers per record
 * (start xyz, end xyz, normal_a xyz, normal_b xyz, label), '#' starts a comment, blank
 * lines skipped; normals normalised on load. Errors: "cannot open edges file: <path>",
 * "edge record R: expected 13 values" / "degenerate edge" / "zero normal" / "normal not
 * perpendicular to edge". */
int pcr_load_edges(pcr_ctx* ctx, const char* path, pcr_edges** out);
void pcr_free_edges(pcr_edges* edges);

/* The file-level fields of RunConfig (pipeline.hpp:12-32) that run_pipeline_on_scene
 * does not take. NULL or "" means "not given", as the reference's empty strings. */
typedef struct pcr_run_files {
  const char* scene_path;  /* PLY point cloud */
  const char* edges_path;  /* edges file */
  const char* output_path; /* paths JSONL */
  const double* tx_position; /* n_tx*3; ids assigned 0..n_tx-1 in order */
  uint32_t n_tx;
  const double* rx_position; /* n_rx*3; ids 0..n_rx-1 */
  uint32_t n_rx;
} pcr_run_files;
/* run_pipeline (pipeline.hpp:63-64; pipeline.cpp:214-247): load (PLY straight to the
 * device + edges) -> run_pipeline_on_scene -> write the paths JSONL when output_path is
 * given. Timings gain "load" first and "write" last; load and write failures carry the
 * "load: " / "write: " prefixes. */
int pcr_run_pipeline(pcr_ctx* ctx, const pcr_run_files* files, const pcr_run_config* config, pcr_summary** out);

/* ---- sharded pipeline: one process per GPU ----------------------------- */
/* run_pipeline_on_scene split across n_shards contexts (one per GPU). The reference
 * parallelises the same loop over initial hits (tracer.cpp:476-533, parallel_for) and
 * refines candidates independently (pipeline.cpp:148-187); the split is exact:
 *   1. pcr_shard_trace: validate + build_grid + transmission_phase (full, on every
 *      shard), then propagate over the initial hits t = shard (mod n_shards) of every
 *      TX with this shard's own first-kappa (a superset of its share of the global
 *      one). Rows: n_rows records of row_bytes (DFS key, group hash, candidate).
 *   2. pcr_shard_rows copies them into caller device memory; the caller all-gathers
 *      every shard's rows (e.g. an NCCL all-gather of a byte tensor).
 *   3. pcr_shard_refine: global kappa over all rows (any concatenation order) -> the
 *      reference's candidate list, identical on every shard; refine candidates
 *      i = shard (mod n_shards). pcr_shard_outcomes copies the n_out outcome rows.
 *   4. pcr_shard_stats returns this shard's work counters; the caller sums them over
 *      shards and gathers every shard's outcome rows to one shard, whose
 *      pcr_shard_finish produces the RunSummary of the unsharded run (same counts,
 *      same exact paths in the same order; timings are this shard's).
 * Device pointers are in the context's device memory; rows are plain bytes. */
typedef struct pcr_shard_stats {
  uint64_t cone_traces, visibility_tests, walk_cells, walk_ies; /* propagation of the shard */
  uint64_t refine_iterations, refine_trials, refine_marches;    /* refinement of the shard */
  uint64_t libm_unresolved, refine_trial_nodes, refine_iter_nodes;
} pcr_shard_stats;
int pcr_shard_trace(pcr_ctx* ctx, const pcr_scene* scene, const pcr_run_config* config, uint32_t shard,
                    uint32_t n_shards, uint64_t* n_rows, uint64_t* row_bytes);
/* pcr_shard_trace on a grid the caller replicated (NCCL broadcast of one part, or the
 * sharded build's all-gathered parts: pcr_grid_assemble); the grid must outlive the
 * context's shard calls */
int pcr_shard_trace_grid(pcr_ctx* ctx, const pcr_scene* scene, const pcr_grid* grid, const pcr_run_config* config,
                         uint32_t shard, uint32_t n_shards, uint64_t* n_rows, uint64_t* row_bytes);
int pcr_shard_rows(pcr_ctx* ctx, void* dst_device);
int pcr_shard_refine(pcr_ctx* ctx, const pcr_scene* scene, const void* rows_device, uint64_t n_rows,
                     uint64_t* n_out, uint64_t* out_row_bytes);
int pcr_shard_outcomes(pcr_ctx* ctx, void* dst_device);
int pcr_shard_stats_get(pcr_ctx* ctx, pcr_shard_stats* out);
int pcr_shard_finish(pcr_ctx* ctx, const void* outcome_rows_device, uint64_t n_rows,
                     const pcr_shard_stats* totals, pcr_summary** out);

/* ---- instrumentation (no reference counterpart) ------------------------------------ */
/* cudaStream_t the context launches on, as an opaque pointer (for caller-side events) */
void* pcr_stream(pcr_ctx* ctx);
/* per-kernel CUDA-event timing of subsequent calls: 1 every kernel, 2 only the refine
 * kernel (one launch per refine call: no events around the many small trace launches
 * inside a timed region), 0 disables */
int pcr_set_profiling(pcr_ctx* ctx, int on);
/* accumulated per-kernel totals since the last reset; returns the number of entries
 * (at most cap); names are NUL-terminated, 32 bytes each. reset != 0 clears them. */
int pcr_kernel_times(pcr_ctx* ctx, char (*names)[32], double* ms, uint64_t* launches, int cap, int reset);

/* measured non-FMA FP64 throughput of this device (TFLOP/s), the refinement roofline */
int pcr_fp64_probe(pcr_ctx* ctx, double* tflops);

/* the device exp() used by the non-planar SDF (estimate_surface), on host arrays:
 * a parity hook — it equals the host libm's exp() bit for bit */
int pcr_libm_exp_batch(pcr_ctx* ctx, const double* x, double* y, uint64_t n);

/* config_hash (pipeline.hpp:39; pipeline.cpp:89-97) */
uint64_t pcr_config_hash(const pcr_run_config* config);
void pcr_run_config_defaults(pcr_run_config* config);

void pcr_free_paths(pcr_paths* p);
void pcr_free_initial_hits(pcr_initial_hits* h);
void pcr_free_outcomes(pcr_outcomes* o);
void pcr_free_summary(pcr_summary* s);
void pcr_free_receptions(pcr_receptions* r);

#ifdef __cplusplus
}
#endif
#endif /* PCRAY_B200_H */
