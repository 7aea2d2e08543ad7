// io.cu — the data formats either side of the hot path:
//
// * point-cloud ingest (load_point_cloud, proj/src/io.cpp:40-158) straight into the
//   device-resident Scene: the header is parsed on the host with the reference's
//   rules and error texts; binary_little_endian vertex data is streamed in chunks
//   through two pinned buffers (read chunk k+1 while chunk k is copied and decoded)
//   and a decode kernel picks x, y, z, nx, ny, nz (float32 -> FP64, exact) and label
//   out of each row at the header's property offsets, skipping unknown properties;
//   ascii data is parsed on the host as the reference does (istream >> double).
// * the paths JSONL writer (write_paths, proj/src/io.cpp:317-349): same header line,
//   same field order, %.9g numbers, records in the order given.
// * the edges file (load_edges, proj/src/io.cpp:191-229) and the file-level pipeline
//   run (run_pipeline, proj/src/pipeline.cpp:214-247) that ties the three together.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>

#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include <algorithm>

#include "exact.cuh"
#include "host_alloc.hpp"
#include "pipeline.hpp"

namespace pcr {

namespace {

// ---- PLY header -------------------------------------------------------------------
// A PLY header (Turk's format): the magic line "ply", one format line, then
// `keyword args...` lines up to "end_header". Only the vertex element is read; its
// scalar properties give the byte layout of a binary row (or the value order of an
// ascii row). Errors carry the texts and 1-based line numbers load_point_cloud
// reports (io.cpp:40-122), since callers and tests match them.

// byte sizes of the PLY scalar types, by every name the format allows
struct PlyType {
  const char* name;
  uint32_t bytes;
};
constexpr PlyType kPlyTypes[] = {
    {"char", 1},  {"int8", 1},   {"uchar", 1},  {"uint8", 1},   {"short", 2},   {"int16", 2},
    {"ushort", 2}, {"uint16", 2}, {"int", 4},    {"int32", 4},   {"uint", 4},    {"uint32", 4},
    {"float", 4}, {"float32", 4}, {"double", 8}, {"float64", 8},
};

struct PlyProp {
  std::string type, name;
  size_t offset = 0;
};

struct PlyHeader {
  bool binary = false;
  size_t vertex_count = 0, stride = 0;
  std::vector<PlyProp> props;
  int idx[7];  // x y z nx ny nz label
};

// whitespace-separated words of a header line
std::vector<std::string> split_words(const std::string& line) {
  std::vector<std::string> w;
  size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
    const size_t b = i;
    while (i < line.size() && !std::isspace(static_cast<unsigned char>(line[i]))) ++i;
    if (i > b) w.emplace_back(line, b, i - b);
  }
  return w;
}

// decimal integer at the start of `word` (optional sign, then digits; trailing
// characters ignored, as a formatted stream read stops there); false if none or out
// of range
bool leading_integer(const std::string& word, long long& v) {
  errno = 0;
  char* end = nullptr;
  const char* b = word.c_str();
  if (*b != '+' && *b != '-' && !std::isdigit(static_cast<unsigned char>(*b))) return false;
  v = std::strtoll(b, &end, 10);
  return end != b && errno != ERANGE;
}

class PlyHeaderReader {
 public:
  explicit PlyHeaderReader(std::istream& in) : in_(in) {}

  PlyHeader read() {
    if (line() != "ply") fail("expected 'ply' magic");
    const std::string& fmt = line();
    if (fmt == "format ascii 1.0")
      h_.binary = false;
    else if (fmt == "format binary_little_endian 1.0")
      h_.binary = true;
    else
      fail("unsupported format '" + fmt + "'");
    for (;;) {
      const std::vector<std::string> w = split_words(line());
      if (w.empty() || w[0] == "comment" || w[0] == "obj_info") continue;
      if (w[0] == "end_header") break;
      if (w[0] == "element")
        element(w);
      else if (w[0] == "property")
        property(w);
      else
        fail("unknown header keyword '" + w[0] + "'");
    }
    if (!vertex_seen_) fail("no vertex element");
    static const char* const kRequired[7] = {"x", "y", "z", "nx", "ny", "nz", "label"};
    for (int r = 0; r < 7; ++r) {
      int found = -1;  // a repeated name: the last declaration is the one read
      for (int i = static_cast<int>(h_.props.size()) - 1; i >= 0 && found < 0; --i)
        if (h_.props[i].name == kRequired[r]) found = i;
      if (found < 0) throw Error(PCR_ERR_RUNTIME, std::string("missing field: ") + kRequired[r]);
      const std::string& t = h_.props[found].type;
      const bool is_f32 = t == "float" || t == "float32", is_u32 = t == "uint" || t == "uint32";
      if (r < 6 && !is_f32) throw Error(PCR_ERR_RUNTIME, std::string("field ") + kRequired[r] + " must be float32");
      if (r == 6 && !is_u32) throw Error(PCR_ERR_RUNTIME, "field label must be uint32");
      h_.idx[r] = found;
    }
    return h_;
  }

 private:
  // "element <name> <count>": only the vertex element is kept; any element with rows
  // declared before it would have to be skipped in the body, which is not supported
  void element(const std::vector<std::string>& w) {
    long long count = -1;
    if (w.size() < 3 || !leading_integer(w[2], count) || count < 0) fail("malformed element declaration");
    in_vertex_ = w[1] == "vertex";
    if (in_vertex_) {
      if (vertex_seen_) fail("duplicate vertex element");
      vertex_seen_ = true;
      h_.vertex_count = static_cast<size_t>(count);
    } else if (!vertex_seen_ && count > 0) {
      fail("element '" + w[1] + "' precedes vertex data");
    }
  }
  // "property <type> <name>" inside the vertex element: appended to the row layout
  void property(const std::vector<std::string>& w) {
    if (!in_vertex_) return;
    const std::string type = w.size() > 1 ? w[1] : std::string();
    if (type == "list") fail("list property in vertex element");
    if (w.size() < 3) fail("malformed property declaration");
    uint32_t bytes = 0;
    for (const PlyType& t : kPlyTypes)
      if (type == t.name) bytes = t.bytes;
    if (!bytes) fail("unknown property type '" + type + "'");
    h_.props.push_back(PlyProp{type, w[2], h_.stride});
    h_.stride += bytes;
  }
  // the next header line (CR of a CRLF file dropped); running out is an error on the
  // line after the last one read
  const std::string& line() {
    if (!std::getline(in_, cur_)) {
      ++n_;
      fail("unexpected end of header");
    }
    ++n_;
    if (!cur_.empty() && cur_.back() == '\r') cur_.pop_back();
    return cur_;
  }
  [[noreturn]] void fail(const std::string& what) const {
    throw Error(PCR_ERR_RUNTIME, "parse error at line " + std::to_string(n_) + ": " + what);
  }

  std::istream& in_;
  std::string cur_;
  int n_ = 0;
  bool in_vertex_ = false, vertex_seen_ = false;
  PlyHeader h_;
};

PlyHeader parse_header(std::istream& in) { return PlyHeaderReader(in).read(); }

struct RowLayout {
  uint32_t stride;
  uint32_t off[7];
};

// One thread per vertex row: float32 fields widened to FP64 (exact), label as is.
__global__ void ply_decode_kernel(const uint8_t* __restrict__ rows, uint64_t n, RowLayout L, uint64_t first,
                                  double* __restrict__ pos, double* __restrict__ nrm, uint32_t* __restrict__ label) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t* r = rows + i * L.stride;
  float f[6];
  for (int k = 0; k < 6; ++k) memcpy(&f[k], r + L.off[k], 4);
  uint32_t lab;
  memcpy(&lab, r + L.off[6], 4);
  const uint64_t v = first + i;
  pos[3 * v] = f[0];
  pos[3 * v + 1] = f[1];
  pos[3 * v + 2] = f[2];
  nrm[3 * v] = f[3];
  nrm[3 * v + 1] = f[4];
  nrm[3 * v + 2] = f[5];
  label[v] = lab;
}

struct Pinned {
  uint8_t* p = nullptr;
  explicit Pinned(size_t n) {
    if (cudaMallocHost(&p, n ? n : 1) != cudaSuccess) throw Error(PCR_ERR_NOMEM, "cudaMallocHost failed");
  }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

// The non-point parts of the scene (edges, radios, frequency) as upload_scene does.
void upload_rest(Ctx& ctx, const pcr_scene_desc& d, SceneDev& S) {
  cudaStream_t s = ctx.stream;
  S.n_edges = d.n_edges;
  S.h_edges.assign(d.edge_geometry, d.edge_geometry + 12ull * d.n_edges);
  S.h_edge_label.assign(d.edge_label, d.edge_label + d.n_edges);
  S.edges.alloc(12ull * d.n_edges + 12, s);
  S.edge_label.alloc(d.n_edges + 1ull, s);
  h2d(S.edges.get(), S.h_edges.data(), S.h_edges.size(), s);
  h2d(S.edge_label.get(), S.h_edge_label.data(), S.h_edge_label.size(), s);
  S.h_tx.assign(d.tx_position, d.tx_position + 3ull * d.n_tx);
  S.h_tx_id.assign(d.tx_id, d.tx_id + d.n_tx);
  S.h_rx.assign(d.rx_position, d.rx_position + 3ull * d.n_rx);
  S.h_rx_id.assign(d.rx_id, d.rx_id + d.n_rx);
  S.rx_pos.alloc(3ull * d.n_rx + 3, s);
  S.rx_id.alloc(d.n_rx + 1ull, s);
  h2d(S.rx_pos.get(), S.h_rx.data(), S.h_rx.size(), s);
  h2d(S.rx_id.get(), S.h_rx_id.data(), S.h_rx_id.size(), s);
  S.carrier_frequency_hz = d.carrier_frequency_hz;
}

std::string fmt9(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.9g", v);
  return buf;
}

}  // namespace

void api_scene_load_ply(Ctx& ctx, const char* path, const pcr_scene_desc& rest, SceneDev& S) {
  cudaStream_t s = ctx.stream;
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(PCR_ERR_RUNTIME, std::string("cannot open point cloud file: ") + path);
  const PlyHeader h = parse_header(in);
  const size_t n = h.vertex_count;
  S.n_points = n;
  S.pos.alloc(3 * n + 3, s);
  S.nrm.alloc(3 * n + 3, s);
  S.label.alloc(n + 1, s);
  if (h.binary) {
    RowLayout L;
    L.stride = static_cast<uint32_t>(h.stride);
    for (int r = 0; r < 7; ++r) L.off[r] = static_cast<uint32_t>(h.props[h.idx[r]].offset);
    // chunks of whole rows, double-buffered: the file read of chunk k+1 overlaps the
    // copy + decode of chunk k
    const size_t rows_per_chunk = std::max<size_t>(1, (size_t(64) << 20) / std::max<size_t>(1, h.stride));
    const size_t chunk_bytes = rows_per_chunk * h.stride;
    Pinned host[2] = {Pinned(chunk_bytes), Pinned(chunk_bytes)};
    DBuf<uint8_t> dev[2];
    dev[0].alloc(chunk_bytes, s);
    dev[1].alloc(chunk_bytes, s);
    cudaEvent_t done[2];
    PCR_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    PCR_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    bool pending[2] = {false, false};
    size_t v = 0;
    int b = 0;
    try {
      while (v < n) {
        const size_t rows = std::min(rows_per_chunk, n - v);
        if (pending[b]) PCR_CUDA(cudaEventSynchronize(done[b]));  // buffer b is free again
        in.read(reinterpret_cast<char*>(host[b].p), static_cast<std::streamsize>(rows * h.stride));
        const size_t got = static_cast<size_t>(in.gcount());
        if (got < rows * h.stride)
          throw Error(PCR_ERR_RUNTIME, "truncated vertex data at record " + std::to_string(v + got / h.stride));
        PCR_CUDA(cudaMemcpyAsync(dev[b].get(), host[b].p, rows * h.stride, cudaMemcpyHostToDevice, s));
        g_h2d_bytes += rows * h.stride;
        count_launch();
        ply_decode_kernel<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(
            dev[b].get(), rows, L, v, S.pos.get(), S.nrm.get(), S.label.get());
        PCR_LAUNCH_CHECK();
        PCR_CUDA(cudaEventRecord(done[b], s));
        pending[b] = true;
        v += rows;
        b ^= 1;
      }
      stream_wait(s);
    } catch (...) {
      cudaStreamSynchronize(s);
      cudaEventDestroy(done[0]);
      cudaEventDestroy(done[1]);
      throw;
    }
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
  } else {
    // ascii: every property parsed as a double in declaration order (io.cpp:139-155)
    std::vector<double> pos(3 * n), nrm(3 * n), values(h.props.size());
    std::vector<uint32_t> lab(n);
    std::string line;
    for (size_t v = 0; v < n; ++v) {
      if (!std::getline(in, line)) throw Error(PCR_ERR_RUNTIME, "truncated vertex data at record " + std::to_string(v));
      std::istringstream iss(line);
      for (size_t i = 0; i < h.props.size(); ++i)
        if (!(iss >> values[i])) throw Error(PCR_ERR_RUNTIME, "malformed vertex data at record " + std::to_string(v));
      for (int a = 0; a < 3; ++a) {
        pos[3 * v + a] = values[h.idx[a]];
        nrm[3 * v + a] = values[h.idx[3 + a]];
      }
      lab[v] = static_cast<uint32_t>(values[h.idx[6]]);
    }
    h2d(S.pos.get(), pos.data(), pos.size(), s);
    h2d(S.nrm.get(), nrm.data(), nrm.size(), s);
    h2d(S.label.get(), lab.data(), lab.size(), s);
  }
  upload_rest(ctx, rest, S);
  stream_wait(s);
}

void api_scene_points(Ctx& ctx, const SceneDev& S, double* pos, double* nrm, uint32_t* label) {
  cudaStream_t s = ctx.stream;
  if (pos) d2h(pos, S.pos.get(), 3 * S.n_points, s);
  if (nrm) d2h(nrm, S.nrm.get(), 3 * S.n_points, s);
  if (label) d2h(label, S.label.get(), S.n_points, s);
  stream_wait(s);
}

// write_paths (io.cpp:317-349): header with the config hash, then one record per path.
void api_write_paths(const char* path, const pcr_paths& p, uint64_t config_hash) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw Error(PCR_ERR_RUNTIME, std::string("cannot write paths file: ") + path);
  char hex[17];
  std::snprintf(hex, sizeof(hex), "%016llx", static_cast<unsigned long long>(config_hash));
  std::string buf;
  buf.reserve(1 << 20);
  buf += "{\"artifact\":\"paths\",\"version\":1,\"config_hash\":\"";
  buf += hex;
  buf += "\"}\n";
  for (uint64_t i = 0; i < p.n; ++i) {
    buf += "{\"tx_id\":" + std::to_string(p.tx_id[i]) + ",\"rx_id\":" + std::to_string(p.rx_id[i]) +
           ",\"delay_s\":" + fmt9(p.delay[i]) + ",\"length_m\":" + fmt9(p.length[i]) +
           ",\"converged\":" + (p.converged[i] ? "true" : "false") + ",\"gradient_norm\":" +
           fmt9(p.gradient_norm[i]) + ",\"interactions\":[";
    for (uint32_t k = 0; k < p.n_inter[i]; ++k) {
      const size_t j = i * p.stride + k;
      if (k) buf += ",";
      buf += std::string("{\"kind\":\"") + (p.kind[j] == 0 ? "reflection" : "diffraction") + "\",\"position\":[" +
             fmt9(p.position[3 * j]) + "," + fmt9(p.position[3 * j + 1]) + "," + fmt9(p.position[3 * j + 2]) +
             "],\"label\":" + std::to_string(p.label[j]) + "}";
    }
    buf += "]}\n";
    if (buf.size() > (1u << 20)) {
      out.write(buf.data(), static_cast<std::streamsize>(buf.size()));
      buf.clear();
    }
  }
  out.write(buf.data(), static_cast<std::streamsize>(buf.size()));
  if (!out) throw Error(PCR_ERR_RUNTIME, std::string("write failure: ") + path);
}

namespace {

// One line of an edges file: `start(3) end(3) normal_a(3) normal_b(3) label`, anything
// after '#' ignored. Numbers are read as formatted stream extraction reads a double
// (the reference's grammar and rounding), left to right.
enum class EdgeLine { kSkip, kShort, kRecord };

EdgeLine read_edge_line(std::string text, double v[13]) {
  text.resize(std::min(text.size(), text.find('#')));
  std::istringstream fields(text);
  int got = 0;
  while (got < 13 && fields >> v[got]) ++got;
  // a line whose first field is not a number carries no record (blank, comment, prose)
  return got == 0 ? EdgeLine::kSkip : got < 13 ? EdgeLine::kShort : EdgeLine::kRecord;
}

// The record's geometry checks (DiffractionEdge invariants, io.cpp:209-222): a
// non-degenerate segment, non-zero normals, and after normalisation both normals
// perpendicular to the edge direction within 1e-3. Normalises v[6..11] in place;
// returns the defect or nullptr.
const char* edge_defect(double v[13]) {
  const V3 a{v[0], v[1], v[2]}, b{v[3], v[4], v[5]};
  V3 na{v[6], v[7], v[8]}, nb{v[9], v[10], v[11]};
  if (norm(b - a) < 1e-12) return "degenerate edge";
  if (norm(na) < 1e-12 || norm(nb) < 1e-12) return "zero normal";
  na = normalized(na);
  nb = normalized(nb);
  const V3 w = normalized(b - a);
  if (std::abs(dot(w, na)) > 1e-3 || std::abs(dot(w, nb)) > 1e-3) return "normal not perpendicular to edge";
  const double n6[6] = {na.x, na.y, na.z, nb.x, nb.y, nb.z};
  std::copy(n6, n6 + 6, v + 6);
  return nullptr;
}

}  // namespace

// load_edges (io.cpp:191-229): geometry rows (start, end, unit normal_a, unit
// normal_b) and labels; the n-th accepted record is "edge record n" in errors.
void api_load_edges(const char* path, std::vector<double>& geom, std::vector<uint32_t>& label) {
  std::ifstream in(path);
  if (!in) throw Error(PCR_ERR_RUNTIME, std::string("cannot open edges file: ") + path);
  geom.clear();
  label.clear();
  std::string text;
  while (std::getline(in, text)) {
    double v[13];
    const EdgeLine kind = read_edge_line(text, v);
    if (kind == EdgeLine::kSkip) continue;
    const char* defect = kind == EdgeLine::kShort ? "expected 13 values" : edge_defect(v);
    if (defect) throw Error(PCR_ERR_RUNTIME, "edge record " + std::to_string(label.size()) + ": " + defect);
    geom.insert(geom.end(), v, v + 12);
    label.push_back(static_cast<uint32_t>(v[12]));
  }
}

// run_pipeline (pipeline.cpp:214-247). The point cloud goes straight to the device
// (api_scene_load_ply); radios get ids 0..n-1 in the order given; the "load" timing
// (points, edges, radios) is inserted before the pipeline's own stages and "write"
// appended after the JSONL is written.
void api_run_pipeline(Ctx& ctx, const pcr_run_files& f, const pcr_run_config& cfg, pcr_summary** out) {
  using Clock = std::chrono::steady_clock;
  auto since = [](Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); };
  const bool has_scene = f.scene_path && *f.scene_path;
  const bool has_edges = f.edges_path && *f.edges_path;
  const bool has_output = f.output_path && *f.output_path;
  auto t0 = Clock::now();
  SceneDev S;
  std::vector<double> eg;
  std::vector<uint32_t> el;
  std::vector<uint32_t> tx_id(f.n_tx), rx_id(f.n_rx);
  for (uint32_t i = 0; i < f.n_tx; ++i) tx_id[i] = i;
  for (uint32_t i = 0; i < f.n_rx; ++i) rx_id[i] = i;
  pcr_scene_desc rest{};
  rest.carrier_frequency_hz = cfg.carrier_frequency_hz;
  try {
    if (has_scene) {
      api_scene_load_ply(ctx, f.scene_path, rest, S);
    } else {
      S.n_points = 0;
      S.pos.alloc(3, ctx.stream);
      S.nrm.alloc(3, ctx.stream);
      S.label.alloc(1, ctx.stream);
    }
    if (has_edges) api_load_edges(f.edges_path, eg, el);
  } catch (const std::exception& e) {
    const Error* pe = dynamic_cast<const Error*>(&e);
    throw Error(pe ? pe->code : PCR_ERR_RUNTIME, std::string("load: ") + e.what());
  }
  rest.edge_geometry = eg.data();
  rest.edge_label = el.data();
  rest.n_edges = static_cast<uint32_t>(el.size());
  rest.tx_position = f.tx_position;
  rest.tx_id = tx_id.data();
  rest.n_tx = f.n_tx;
  rest.rx_position = f.rx_position;
  rest.rx_id = rx_id.data();
  rest.n_rx = f.n_rx;
  upload_rest(ctx, rest, S);
  PCR_CUDA(cudaStreamSynchronize(ctx.stream));
  const double load_seconds = since(t0);

  pcr_summary* sum = nullptr;
  api_run_pipeline_device(ctx, S, cfg, &sum);
  struct Guard {
    pcr_summary* s;
    ~Guard() {
      if (s) {
        free_paths_arrays(&s->paths);
        std::free(s);
      }
    }
  } guard{sum};
  if (sum->n_timings < PCR_MAX_STAGES) {
    for (uint32_t t = sum->n_timings; t > 0; --t) {
      std::memcpy(sum->timing_stage[t], sum->timing_stage[t - 1], sizeof(sum->timing_stage[t]));
      sum->timing_seconds[t] = sum->timing_seconds[t - 1];
    }
    std::snprintf(sum->timing_stage[0], sizeof(sum->timing_stage[0]), "load");
    sum->timing_seconds[0] = load_seconds;
    ++sum->n_timings;
  }
  if (has_output) {
    t0 = Clock::now();
    try {
      api_write_paths(f.output_path, sum->paths, sum->hash);
    } catch (const std::exception& e) {
      const Error* pe = dynamic_cast<const Error*>(&e);
      throw Error(pe ? pe->code : PCR_ERR_RUNTIME, std::string("write: ") + e.what());
    }
    if (sum->n_timings < PCR_MAX_STAGES) {
      std::snprintf(sum->timing_stage[sum->n_timings], sizeof(sum->timing_stage[0]), "write");
      sum->timing_seconds[sum->n_timings++] = since(t0);
    }
  }
  *out = sum;
  guard.s = nullptr;
}

}  // namespace pcr
