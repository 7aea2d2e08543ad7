// pcray_mgpu.cpp — the multi-GPU host driver: one process per GPU of one
// node, NCCL over NVLink for every exchange, the B200 library (include/pcray_b200.h)
// for all compute. It replaces the reference's in-process parallel_for loops
// (proj/src/pipeline.cpp:136-187 over TX / candidates, proj/src/tracer.cpp:476-533
// over initial hits) with a split across processes:
//
//   scene     every rank loads the PLY straight into its GPU (pcr_scene_load_ply) + edges
//   grid      --grid broadcast: rank 0 builds the grid, ncclBroadcast of its bytes,
//             every rank assembles it (the north star's "voxel structures replicated by
//             an NCCL broadcast"); --grid sharded: each rank builds the part of its voxel
//             range (pcr_grid_part_build), ncclAllGather of the parts, every rank
//             assembles the whole grid (bit-identical to the unsharded build)
//   trace     pcr_shard_trace_grid: transmission on every rank, propagate over the
//             initial hits t = rank (mod world); candidate rows ncclAllGather'ed
//   refine    pcr_shard_refine: global kappa, candidates i = rank (mod world); outcome
//             rows and the work counters (ncclAllReduce) to rank 0
//   finish    rank 0: pcr_shard_finish (dedup, final order) = the unsharded RunSummary;
//             the paths JSONL when --out is given
//
// Launch: one process per GPU with RANK / WORLD_SIZE / LOCAL_RANK in the environment
// (torchrun, or any launcher that sets them); the NCCL unique id travels through the
// file named by PCRAY_NCCL_ID (default /tmp/pcray_nccl_<MASTER_PORT>.id), which works
// for the single-node scope. Prints one JSON line on rank 0: counts, per-stage device
// seconds (max over ranks), the per-rank trace / refine split.
//
//   pcray_mgpu --ply scene.ply --radios radios.txt [--edges e.txt] [--out paths.jsonl]
//              [--grid broadcast|sharded] [--max-interactions 4] [--max-diffractions 1]
//              [--kappa 100] [--voxel 0.5] [--division 2] [--reps 1]
#include <cuda_runtime.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "pcray_b200.h"

namespace {

[[noreturn]] void die(const std::string& m) { throw std::runtime_error(m); }

#define NCCL_OK(x)                                                                    \
  do {                                                                                \
    const ncclResult_t r_ = (x);                                                      \
    if (r_ != ncclSuccess) die(std::string("nccl ") + #x + ": " + ncclGetErrorString(r_)); \
  } while (0)
#define CUDA_OK(x)                                                                    \
  do {                                                                                \
    const cudaError_t r_ = (x);                                                       \
    if (r_ != cudaSuccess) die(std::string("cuda ") + #x + ": " + cudaGetErrorString(r_)); \
  } while (0)

int env_int(const char* k, int d) {
  const char* v = std::getenv(k);
  return v ? std::atoi(v) : d;
}

struct Args {
  std::string ply, edges, radios, out, grid = "sharded";
  int reps = 1;
  pcr_run_config cfg{};
};

Args parse(int argc, char** argv) {
  Args a;
  pcr_run_config_defaults(&a.cfg);
  for (int i = 1; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) die("missing value for " + k);
      return argv[++i];
    };
    if (k == "--ply") a.ply = val();
    else if (k == "--edges") a.edges = val();
    else if (k == "--radios") a.radios = val();
    else if (k == "--out") a.out = val();
    else if (k == "--grid") a.grid = val();
    else if (k == "--reps") a.reps = std::stoi(val());
    else if (k == "--max-interactions") a.cfg.max_interactions = std::stoi(val());
    else if (k == "--max-diffractions") a.cfg.max_diffractions = std::stoi(val());
    else if (k == "--kappa") a.cfg.kappa = std::stoi(val());
    else if (k == "--voxel") a.cfg.voxel_size_m = std::stod(val());
    else if (k == "--division") a.cfg.division_factor = std::stoi(val());
    else die("unknown argument " + k);
  }
  if (a.ply.empty() || a.radios.empty()) die("--ply and --radios are required");
  if (a.grid != "broadcast" && a.grid != "sharded") die("--grid is broadcast or sharded");
  return a;
}

// radios file: "tx x y z" / "rx x y z" per line, '#' comments; ids 0..n-1 in order
// (as run_pipeline assigns them, proj/src/pipeline.cpp:224-231)
void load_radios(const std::string& path, std::vector<double>& tx, std::vector<double>& rx) {
  std::ifstream in(path);
  if (!in) die("cannot open radios file: " + path);
  std::string line;
  while (std::getline(in, line)) {
    line.resize(std::min(line.size(), line.find('#')));
    std::istringstream f(line);
    std::string kind;
    double p[3];
    if (!(f >> kind)) continue;
    if (!(f >> p[0] >> p[1] >> p[2]) || (kind != "tx" && kind != "rx")) die("bad radios line: " + line);
    (kind == "tx" ? tx : rx).insert((kind == "tx" ? tx : rx).end(), p, p + 3);
  }
}

struct Lib {
  pcr_ctx* ctx = nullptr;
  void check(int rc) const {
    if (rc != PCR_OK) die(pcr_last_error(ctx));
  }
};

struct Comm {
  ncclComm_t c;
  int rank, world;
  cudaStream_t s;
};

ncclUniqueId bootstrap_id(int rank) {
  std::string path = std::getenv("PCRAY_NCCL_ID") ? std::getenv("PCRAY_NCCL_ID")
                                                  : "/tmp/pcray_nccl_" + std::to_string(env_int("MASTER_PORT", 29500)) + ".id";
  ncclUniqueId id;
  if (rank == 0) {
    NCCL_OK(ncclGetUniqueId(&id));
    const std::string tmp = path + ".tmp";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f || std::fwrite(&id, sizeof(id), 1, f) != 1) die("cannot write " + tmp);
    std::fclose(f);
    if (std::rename(tmp.c_str(), path.c_str()) != 0) die("cannot publish " + path);
  } else {
    for (int t = 0;; ++t) {
      FILE* f = std::fopen(path.c_str(), "rb");
      if (f && std::fread(&id, sizeof(id), 1, f) == 1) {
        std::fclose(f);
        break;
      }
      if (f) std::fclose(f);
      if (t > 6000) die("timed out waiting for " + path);
      usleep(10000);
    }
  }
  return id;
}

// variable-size all-gather of device bytes: sizes first, then padded blocks; the result
// is compacted so rank r's bytes start at offset[r]
std::vector<uint64_t> all_gather_bytes(const Comm& cm, const void* mine, uint64_t n, void** out, uint64_t* total) {
  uint64_t *d_sz, *d_all;
  CUDA_OK(cudaMalloc(&d_sz, 8));
  CUDA_OK(cudaMalloc(&d_all, 8ull * cm.world));
  CUDA_OK(cudaMemcpyAsync(d_sz, &n, 8, cudaMemcpyHostToDevice, cm.s));
  NCCL_OK(ncclAllGather(d_sz, d_all, 1, ncclUint64, cm.c, cm.s));
  std::vector<uint64_t> sizes(cm.world);
  CUDA_OK(cudaMemcpyAsync(sizes.data(), d_all, 8ull * cm.world, cudaMemcpyDeviceToHost, cm.s));
  CUDA_OK(cudaStreamSynchronize(cm.s));
  CUDA_OK(cudaFree(d_sz));
  CUDA_OK(cudaFree(d_all));
  const uint64_t cap = std::max<uint64_t>(1, *std::max_element(sizes.begin(), sizes.end()));
  uint8_t *pad, *all, *res;
  CUDA_OK(cudaMalloc(&pad, cap));
  CUDA_OK(cudaMalloc(&all, cap * cm.world));
  if (n) CUDA_OK(cudaMemcpyAsync(pad, mine, n, cudaMemcpyDeviceToDevice, cm.s));
  NCCL_OK(ncclAllGather(pad, all, cap, ncclUint8, cm.c, cm.s));
  std::vector<uint64_t> off(cm.world);
  uint64_t t = 0;
  for (int r = 0; r < cm.world; ++r) {
    off[r] = t;
    t += sizes[r];
  }
  CUDA_OK(cudaMalloc(&res, std::max<uint64_t>(1, t)));
  for (int r = 0; r < cm.world; ++r)
    if (sizes[r]) CUDA_OK(cudaMemcpyAsync(res + off[r], all + cap * r, sizes[r], cudaMemcpyDeviceToDevice, cm.s));
  CUDA_OK(cudaStreamSynchronize(cm.s));
  CUDA_OK(cudaFree(pad));
  CUDA_OK(cudaFree(all));
  *out = res;
  *total = t;
  sizes.insert(sizes.end(), off.begin(), off.end());  // [sizes..., offsets...]
  return sizes;
}

double max_over_ranks(const Comm& cm, double v) {
  double* d;
  CUDA_OK(cudaMalloc(&d, sizeof(double)));
  CUDA_OK(cudaMemcpyAsync(d, &v, sizeof(double), cudaMemcpyHostToDevice, cm.s));
  NCCL_OK(ncclAllReduce(d, d, 1, ncclFloat64, ncclMax, cm.c, cm.s));
  CUDA_OK(cudaMemcpyAsync(&v, d, sizeof(double), cudaMemcpyDeviceToHost, cm.s));
  CUDA_OK(cudaStreamSynchronize(cm.s));
  CUDA_OK(cudaFree(d));
  return v;
}

struct Timer {  // device time on the library's stream
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  double stop() {
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms * 1e-3;
  }
};

int run(int argc, char** argv) {
  const Args A = parse(argc, argv);
  const int rank = env_int("RANK", 0), world = env_int("WORLD_SIZE", 1), local = env_int("LOCAL_RANK", 0);
  CUDA_OK(cudaSetDevice(local));
  Lib L;
  if (pcr_create(local, &L.ctx) != PCR_OK) die("pcr_create failed (no CUDA device)");
  Comm cm{nullptr, rank, world, static_cast<cudaStream_t>(pcr_stream(L.ctx))};
  const ncclUniqueId id = bootstrap_id(rank);
  NCCL_OK(ncclCommInitRank(&cm.c, world, id, rank));

  // scene: points straight to this GPU; edges and radios from their files
  std::vector<double> tx, rx;
  load_radios(A.radios, tx, rx);
  std::vector<uint32_t> tx_id(tx.size() / 3), rx_id(rx.size() / 3);
  for (size_t i = 0; i < tx_id.size(); ++i) tx_id[i] = static_cast<uint32_t>(i);
  for (size_t i = 0; i < rx_id.size(); ++i) rx_id[i] = static_cast<uint32_t>(i);
  pcr_edges* edges = nullptr;
  if (!A.edges.empty()) L.check(pcr_load_edges(L.ctx, A.edges.c_str(), &edges));
  pcr_scene_desc rest{};
  rest.edge_geometry = edges ? edges->geometry : nullptr;
  rest.edge_label = edges ? edges->label : nullptr;
  rest.n_edges = edges ? edges->n : 0;
  rest.tx_position = tx.data();
  rest.tx_id = tx_id.data();
  rest.n_tx = static_cast<uint32_t>(tx_id.size());
  rest.rx_position = rx.data();
  rest.rx_id = rx_id.data();
  rest.n_rx = static_cast<uint32_t>(rx_id.size());
  rest.carrier_frequency_hz = A.cfg.carrier_frequency_hz;
  pcr_scene* scene = nullptr;
  L.check(pcr_scene_load_ply(L.ctx, A.ply.c_str(), &rest, &scene));
  const pcr_voxel_params vp{A.cfg.voxel_size_m, A.cfg.division_factor, uint64_t(1) << 27};

  double t_grid = 0, t_trace = 0, t_refine = 0, t_finish = 0, t_step = 0;
  pcr_summary* S = nullptr;
  uint64_t my_rows = 0, my_out = 0;
  for (int rep = 0; rep < A.reps; ++rep) {
    if (S) pcr_free_summary(S), S = nullptr;
    CUDA_OK(cudaStreamSynchronize(cm.s));
    Timer step(cm.s);
    // ---- grid
    Timer tg(cm.s);
    pcr_grid* grid = nullptr;
    {
      const bool bcast = A.grid == "broadcast";
      uint64_t nb = 0;
      if (!bcast || rank == 0) L.check(pcr_grid_part_build(L.ctx, scene, &vp, bcast ? 0 : rank, bcast ? 1 : world, &nb));
      void* parts = nullptr;
      std::vector<uint64_t> off, sz;
      if (bcast) {
        uint64_t* d;
        CUDA_OK(cudaMalloc(&d, 8));
        CUDA_OK(cudaMemcpyAsync(d, &nb, 8, cudaMemcpyHostToDevice, cm.s));
        NCCL_OK(ncclBroadcast(d, d, 1, ncclUint64, 0, cm.c, cm.s));
        CUDA_OK(cudaMemcpyAsync(&nb, d, 8, cudaMemcpyDeviceToHost, cm.s));
        CUDA_OK(cudaStreamSynchronize(cm.s));
        CUDA_OK(cudaFree(d));
        CUDA_OK(cudaMalloc(&parts, nb));
        if (rank == 0) L.check(pcr_grid_part_copy(L.ctx, parts));
        NCCL_OK(ncclBroadcast(parts, parts, nb, ncclUint8, 0, cm.c, cm.s));
        off = {0};
        sz = {nb};
      } else {
        void* mine;
        CUDA_OK(cudaMalloc(&mine, std::max<uint64_t>(1, nb)));
        L.check(pcr_grid_part_copy(L.ctx, mine));
        uint64_t total = 0;
        const auto so = all_gather_bytes(cm, mine, nb, &parts, &total);
        CUDA_OK(cudaFree(mine));
        sz.assign(so.begin(), so.begin() + world);
        off.assign(so.begin() + world, so.end());
      }
      CUDA_OK(cudaStreamSynchronize(cm.s));
      L.check(pcr_grid_assemble(L.ctx, parts, off.data(), sz.data(), static_cast<uint32_t>(sz.size()), &grid));
      CUDA_OK(cudaFree(parts));
    }
    t_grid = max_over_ranks(cm, tg.stop());
    // ---- trace: own initial hits, candidate rows to everyone
    Timer tt(cm.s);
    uint64_t n_rows = 0, rb = 0;
    L.check(pcr_shard_trace_grid(L.ctx, scene, grid, &A.cfg, rank, world, &n_rows, &rb));
    my_rows = n_rows;
    void* rows;
    CUDA_OK(cudaMalloc(&rows, std::max<uint64_t>(1, n_rows * rb)));
    if (n_rows) L.check(pcr_shard_rows(L.ctx, rows));
    void* all_rows = nullptr;
    uint64_t all_bytes = 0;
    all_gather_bytes(cm, rows, n_rows * rb, &all_rows, &all_bytes);
    CUDA_OK(cudaFree(rows));
    t_trace = max_over_ranks(cm, tt.stop());
    // ---- refine: global kappa, own candidates; outcome rows + counters to rank 0
    Timer tr(cm.s);
    uint64_t n_out = 0, ob = 0;
    L.check(pcr_shard_refine(L.ctx, scene, all_rows, all_bytes / rb, &n_out, &ob));
    my_out = n_out;
    CUDA_OK(cudaFree(all_rows));
    void* outs;
    CUDA_OK(cudaMalloc(&outs, std::max<uint64_t>(1, n_out * ob)));
    if (n_out) L.check(pcr_shard_outcomes(L.ctx, outs));
    void* all_outs = nullptr;
    uint64_t out_bytes = 0;
    all_gather_bytes(cm, outs, n_out * ob, &all_outs, &out_bytes);
    CUDA_OK(cudaFree(outs));
    pcr_shard_stats st{};
    L.check(pcr_shard_stats_get(L.ctx, &st));
    const int nst = sizeof(st) / sizeof(uint64_t);
    uint64_t* d;
    CUDA_OK(cudaMalloc(&d, sizeof(st)));
    CUDA_OK(cudaMemcpyAsync(d, &st, sizeof(st), cudaMemcpyHostToDevice, cm.s));
    NCCL_OK(ncclAllReduce(d, d, nst, ncclUint64, ncclSum, cm.c, cm.s));
    CUDA_OK(cudaMemcpyAsync(&st, d, sizeof(st), cudaMemcpyDeviceToHost, cm.s));
    CUDA_OK(cudaStreamSynchronize(cm.s));
    CUDA_OK(cudaFree(d));
    t_refine = max_over_ranks(cm, tr.stop());
    // ---- finish on rank 0
    Timer tf(cm.s);
    if (rank == 0) L.check(pcr_shard_finish(L.ctx, all_outs, out_bytes / ob, &st, &S));
    CUDA_OK(cudaFree(all_outs));
    t_finish = max_over_ranks(cm, tf.stop());
    t_step = max_over_ranks(cm, step.stop());
    pcr_grid_free(grid);
  }
  // per-rank split of the work (load balance of the cyclic split)
  std::vector<double> mine = {static_cast<double>(my_rows), static_cast<double>(my_out)};
  double *d, *all;
  CUDA_OK(cudaMalloc(&d, 2 * sizeof(double)));
  CUDA_OK(cudaMalloc(&all, 2 * sizeof(double) * world));
  CUDA_OK(cudaMemcpyAsync(d, mine.data(), 2 * sizeof(double), cudaMemcpyHostToDevice, cm.s));
  NCCL_OK(ncclAllGather(d, all, 2, ncclFloat64, cm.c, cm.s));
  std::vector<double> split(2 * world);
  CUDA_OK(cudaMemcpyAsync(split.data(), all, split.size() * sizeof(double), cudaMemcpyDeviceToHost, cm.s));
  CUDA_OK(cudaStreamSynchronize(cm.s));
  if (rank == 0) {
    if (!A.out.empty()) L.check(pcr_write_paths(L.ctx, A.out.c_str(), &S->paths, S->hash));
    std::printf("{\"world\": %d, \"grid\": \"%s\", \"point_count\": %llu, \"ie_count\": %llu, \"coarse_paths\": %llu, "
                "\"refined_paths\": %llu, \"exact_paths\": %llu, \"rejected\": [%llu, %llu, %llu, %llu], "
                "\"cone_traces\": %llu, \"transmission_rays\": %llu, \"hash\": %llu, "
                "\"seconds\": {\"grid\": %.6f, \"trace\": %.6f, \"refine\": %.6f, \"finish\": %.6f, \"step\": %.6f}, "
                "\"rows_per_rank\": [",
                world, A.grid.c_str(), (unsigned long long)S->point_count, (unsigned long long)S->ie_count,
                (unsigned long long)S->coarse_paths, (unsigned long long)S->refined_paths,
                (unsigned long long)S->exact_paths, (unsigned long long)S->rejected[0],
                (unsigned long long)S->rejected[1], (unsigned long long)S->rejected[2],
                (unsigned long long)S->rejected[3], (unsigned long long)S->cone_traces,
                (unsigned long long)S->transmission_rays, (unsigned long long)S->hash, t_grid, t_trace, t_refine,
                t_finish, t_step);
    for (int r = 0; r < world; ++r) std::printf("%s%.0f", r ? ", " : "", split[2 * r]);
    std::printf("], \"outcomes_per_rank\": [");
    for (int r = 0; r < world; ++r) std::printf("%s%.0f", r ? ", " : "", split[2 * r + 1]);
    std::printf("]}\n");
    std::fflush(stdout);
  }
  if (S) pcr_free_summary(S);
  if (edges) pcr_free_edges(edges);
  pcr_scene_free(scene);
  ncclCommDestroy(cm.c);
  pcr_destroy(L.ctx);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(argc, argv);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "pcray_mgpu: %s\n", e.what());
    return 1;
  }
}
