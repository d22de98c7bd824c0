// tacchi_b200.hpp — header-only C++ mirror of the reference simulator API
// (/root/reference/proj/include/tacchi) over the C-ABI in tacchi_cuda.h.
//
// A caller of the reference swaps
//     #include "tacchi/mpm/engine.hpp"        -> #include "tacchi_b200.hpp"
//     tacchi::mpm::step(state, v, 10)         -> tacchi_b200::mpm::step(state, v, 10)
//     tacchi::sim::capture(state, cfg, obj)   -> tacchi_b200::sim::capture(state, cfg_json, obj)
// and keeps its control flow: the same functions, argument meaning and
// exception classes (errors.hpp:9-39). SimState owns a device handle; its
// particle arrays live in HBM and are copied to host only on request.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tacchi_cuda.h"

namespace tacchi_b200 {

// ---- errors (errors.hpp:9-39) ----------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class GridTooSmall : public Error { public: using Error::Error; };
class EmptyScene : public Error { public: using Error::Error; };
class OutOfGrid : public Error { public: using Error::Error; };
class DegenerateF : public Error { public: using Error::Error; };
class ParseError : public Error { public: using Error::Error; };
class EmptyCloud : public Error { public: using Error::Error; };
class NoSurface : public Error { public: using Error::Error; };
class CropOutOfBounds : public Error { public: using Error::Error; };
class ShapeMismatch : public Error { public: using Error::Error; };
class ConfigError : public Error { public: using Error::Error; };
class IoError : public Error { public: using Error::Error; };
class CudaError : public Error { public: using Error::Error; };
class SessionNotInitialized : public Error { public: using Error::Error; };
class NonMonotonicTime : public Error { public: using Error::Error; };
class ProtocolError : public Error { public: using Error::Error; };
class ManifestMismatch : public Error { public: using Error::Error; };

inline void check(int rc) {
  if (rc == TG_OK) return;
  const std::string m = tg_last_error();
  switch (rc) {
    case TG_ERR_GRID_TOO_SMALL: throw GridTooSmall(m);
    case TG_ERR_EMPTY_SCENE: throw EmptyScene(m);
    case TG_ERR_OUT_OF_GRID: throw OutOfGrid(m);
    case TG_ERR_DEGENERATE_F: throw DegenerateF(m);
    case TG_ERR_CONFIG: throw ConfigError(m);
    case TG_ERR_NO_SURFACE: throw NoSurface(m);
    case TG_ERR_CROP_OUT_OF_BOUNDS: throw CropOutOfBounds(m);
    case TG_ERR_SHAPE_MISMATCH: throw ShapeMismatch(m);
    case TG_ERR_EMPTY_CLOUD: throw EmptyCloud(m);
    case TG_ERR_PARSE: throw ParseError(m);
    case TG_ERR_IO: throw IoError(m);
    case TG_ERR_SESSION_NOT_INITIALIZED: throw SessionNotInitialized(m);
    case TG_ERR_NON_MONOTONIC_TIME: throw NonMonotonicTime(m);
    case TG_ERR_PROTOCOL: throw ProtocolError(m);
    case TG_ERR_MANIFEST_MISMATCH: throw ManifestMismatch(m);
    case TG_ERR_CUDA: throw CudaError(m);
    default: throw Error(m);
  }
}

using Vec3 = std::array<double, 3>;

// ---- render types (depth_map.hpp:11-22, image.hpp:10-23) ----------------
namespace render {
struct DepthMap {
  int width = 0, height = 0;
  double pixel_to_meter = 0.0;
  std::vector<double> values;  // row-major, row = image y
  double at(int row, int col) const { return values[static_cast<size_t>(row) * width + col]; }
};
struct Image8 {
  int width = 0, height = 0;
  std::vector<uint8_t> data;  // interleaved RGB
  uint8_t at(int row, int col, int ch) const {
    return data[(static_cast<size_t>(row) * width + col) * 3 + ch];
  }
};
}  // namespace render

namespace mpm {

struct StepDiagnostics {
  double min_det_f = 1.0;
  double max_speed = 0.0;
};

// mpm::SimState (sim_state.hpp:59-79), device resident.
class SimState {
 public:
  explicit SimState(tg_handle h) : h_(h, &tg_destroy) {}
  tg_handle handle() const { return h_.get(); }
  int64_t size() const { return tg_num_particles(h_.get()); }
  int64_t elastomer_count() const { return tg_num_elastomer(h_.get()); }
  StepDiagnostics diag() const {
    StepDiagnostics d;
    int64_t sc;
    check(tg_diag(h_.get(), &d.min_det_f, &d.max_speed, &sc, nullptr));
    return d;
  }
  int64_t step_count() const {
    int64_t sc;
    check(tg_diag(h_.get(), nullptr, nullptr, &sc, nullptr));
    return sc;
  }
  // Host snapshots in the reference's particle order (row layout).
  void download(std::vector<double>* x, std::vector<double>* v, std::vector<double>* C,
                std::vector<double>* F) const {
    const size_t n = static_cast<size_t>(size());
    if (x) x->resize(3 * n);
    if (v) v->resize(3 * n);
    if (C) C->resize(9 * n);
    if (F) F->resize(9 * n);
    check(tg_download(h_.get(), x ? x->data() : nullptr, v ? v->data() : nullptr,
                      C ? C->data() : nullptr, F ? F->data() : nullptr));
  }
  void upload(const double* x, const double* v, const double* C, const double* F) {
    check(tg_upload(h_.get(), x, v, C, F));
  }
  // ParticleStore::mass / volume0 / tag (reference order).
  void constants(std::vector<double>* mass, std::vector<double>* volume0,
                 std::vector<uint8_t>* tag) const {
    const size_t n = static_cast<size_t>(size());
    if (mass) mass->resize(n);
    if (volume0) volume0->resize(n);
    if (tag) tag->resize(n);
    check(tg_download_constants(h_.get(), mass ? mass->data() : nullptr,
                                volume0 ? volume0->data() : nullptr, tag ? tag->data() : nullptr));
  }
  // Grid::active_lo / active_hi (grid.hpp:25-26).
  std::array<std::array<int, 3>, 2> grid_window() const {
    std::array<std::array<int, 3>, 2> w{};
    check(tg_grid_window(h_.get(), w[0].data(), w[1].data()));
    return w;
  }
  // Grid::mass / momentum / velocity over the node box [lo, hi), k fastest
  // (momentum / velocity: 3 per node). After a step this needs
  // set_keep_grid(true) before stepping (tg_download_grid).
  struct GridBox {
    std::vector<double> mass, momentum, velocity;
  };
  GridBox grid(const std::array<int, 3>& lo, const std::array<int, 3>& hi) const {
    const size_t cnt = static_cast<size_t>(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
    GridBox g;
    g.mass.resize(cnt);
    g.momentum.resize(3 * cnt);
    g.velocity.resize(3 * cnt);
    check(tg_download_grid(h_.get(), lo.data(), hi.data(), g.mass.data(), g.momentum.data(),
                           g.velocity.data()));
    return g;
  }
  void set_keep_grid(bool on) { check(tg_set_keep_grid(h_.get(), on ? 1 : 0)); }

 private:
  std::unique_ptr<tg_sim, void (*)(tg_handle)> h_;
};

// mpm::SceneParams (sim_state.hpp:81-98).
struct SceneParams {
  std::array<int, 3> grid_resolution = {256, 256, 256};
  double grid_edge = 0.033;
  Vec3 grid_origin = {0.0, 0.0, 0.0};
  double youngs_modulus = 1.45e5, poisson_ratio = 0.45, density = 1000.0;
  double dt = 1e-4;
  int fixed_bottom_layers = 2;
  Vec3 gravity = {0.0, 0.0, 0.0};
  double indenter_mass_scale = 80.0;
};

// An elastomer geo::ParticleSet with LatticeMeta (particle_set.hpp:18-30);
// empty positions = make_elastomer_lattice(dims, counts, origin).
struct ElastomerLattice {
  std::array<int, 3> counts = {101, 101, 21};
  Vec3 dims = {0.02, 0.02, 0.004};
  Vec3 origin = {0.0, 0.0, 0.0};
  std::vector<Vec3> positions;
};

// mpm::init_scene (sim_state.hpp:102-104, scene.cpp:28-87).
inline SimState init_scene(const SceneParams& p, const ElastomerLattice& elastomer,
                           const std::vector<Vec3>& indenter,
                           const Vec3& indenter_velocity = {0.0, 0.0, 0.0}, int device = 0) {
  tg_scene_params sp{};
  for (int a = 0; a < 3; ++a) {
    sp.grid_resolution[a] = p.grid_resolution[a];
    sp.grid_origin[a] = p.grid_origin[a];
    sp.gravity[a] = p.gravity[a];
  }
  sp.grid_edge = p.grid_edge;
  sp.youngs_modulus = p.youngs_modulus;
  sp.poisson_ratio = p.poisson_ratio;
  sp.density = p.density;
  sp.dt = p.dt;
  sp.fixed_bottom_layers = p.fixed_bottom_layers;
  sp.indenter_mass_scale = p.indenter_mass_scale;
  tg_lattice lat{};
  for (int a = 0; a < 3; ++a) {
    lat.counts[a] = elastomer.counts[a];
    lat.dims[a] = elastomer.dims[a];
    lat.origin[a] = elastomer.origin[a];
  }
  lat.positions = elastomer.positions.empty() ? nullptr : elastomer.positions.front().data();
  tg_handle h = nullptr;
  check(tg_init_scene(device, &sp, &lat, indenter.empty() ? nullptr : indenter.front().data(),
                      static_cast<int64_t>(indenter.size()), indenter_velocity.data(), &h));
  return SimState(h);
}

// engine.hpp:10-35
inline void zero_grid(SimState& s) { check(tg_phase(s.handle(), TG_PHASE_ZERO_GRID, nullptr)); }
inline void particle_to_grid(SimState& s) {
  check(tg_phase(s.handle(), TG_PHASE_PARTICLE_TO_GRID, nullptr));
}
inline void grid_update(SimState& s) { check(tg_phase(s.handle(), TG_PHASE_GRID_UPDATE, nullptr)); }
inline void grid_to_particle(SimState& s) {
  check(tg_phase(s.handle(), TG_PHASE_GRID_TO_PARTICLE, nullptr));
}
inline void apply_boundary(SimState& s, const Vec3& v) {
  check(tg_phase(s.handle(), TG_PHASE_APPLY_BOUNDARY, v.data()));
}
inline void advect(SimState& s) { check(tg_phase(s.handle(), TG_PHASE_ADVECT, nullptr)); }
inline void step(SimState& s, const Vec3& indenter_velocity, int n_substeps = 1) {
  check(tg_step(s.handle(), indenter_velocity.data(), n_substeps));
}

}  // namespace mpm

namespace sim {

// sim::build_sim(cfg, place_for_press(cfg, indenter_cloud_for(cfg, object), ox, oy))
inline mpm::SimState build_sim(const std::string& config_json, const std::string& object = "",
                               double offset_x = 0.0, double offset_y = 0.0, int device = 0) {
  tg_handle h = nullptr;
  check(tg_build_sim(device, config_json.c_str(), object.c_str(), offset_x, offset_y, &h));
  return mpm::SimState(h);
}

// sim::build_sim(cfg, indenter) (scene_builder.hpp:29-30) with caller-placed
// indenter points (m).
inline mpm::SimState build_sim(const std::string& config_json, const std::vector<Vec3>& indenter,
                               int device = 0) {
  tg_handle h = nullptr;
  check(tg_build_sim_points(device, config_json.c_str(),
                            indenter.empty() ? nullptr : indenter.front().data(),
                            static_cast<int64_t>(indenter.size()), &h));
  return mpm::SimState(h);
}

struct Capture {
  render::DepthMap depth;
  render::Image8 image;
};

// capture's render inputs (lights, RenderParams, alignment_for(object)),
// resolved from the SceneConfig once (scene_config.cpp:70-81) and reused for
// every frame.
struct RenderSetup {
  tg_render r{};
  static RenderSetup from_config(const std::string& config_json, const std::string& object) {
    RenderSetup rs;
    check(tg_render_from_config(config_json.c_str(), object.c_str(), &rs.r));
    return rs;
  }
};

// sim::capture (scene_builder.cpp:80-89) with resolved render inputs.
inline Capture capture(const mpm::SimState& s, const RenderSetup& rs) {
  const tg_render& r = rs.r;
  Capture c;
  c.depth.width = c.image.width = r.width;
  c.depth.height = c.image.height = r.height;
  c.depth.pixel_to_meter = r.pixel_to_meter * r.crop_scale;
  c.depth.values.resize(static_cast<size_t>(r.width) * r.height);
  c.image.data.resize(static_cast<size_t>(r.width) * r.height * 3);
  check(tg_capture(s.handle(), &r, c.depth.values.data(), c.image.data.data()));
  return c;
}

// sim::capture (scene_builder.cpp:80-89)
inline Capture capture(const mpm::SimState& s, const std::string& config_json,
                       const std::string& object) {
  tg_render r;
  check(tg_render_from_config(config_json.c_str(), object.c_str(), &r));
  Capture c;
  c.depth.width = c.image.width = r.width;
  c.depth.height = c.image.height = r.height;
  c.depth.pixel_to_meter = r.pixel_to_meter * r.crop_scale;
  c.depth.values.resize(static_cast<size_t>(r.width) * r.height);
  c.image.data.resize(static_cast<size_t>(r.width) * r.height * 3);
  check(tg_capture(s.handle(), &r, c.depth.values.data(), c.image.data.data()));
  return c;
}

// One Session control step (session.cpp:86 + 42): mpm::step then capture,
// submitted together with one host synchronisation.
inline Capture step_capture(mpm::SimState& s, const Vec3& indenter_velocity, int n_substeps,
                            const std::string& config_json, const std::string& object) {
  tg_render r;
  check(tg_render_from_config(config_json.c_str(), object.c_str(), &r));
  Capture c;
  c.depth.width = c.image.width = r.width;
  c.depth.height = c.image.height = r.height;
  c.depth.pixel_to_meter = r.pixel_to_meter * r.crop_scale;
  c.depth.values.resize(static_cast<size_t>(r.width) * r.height);
  c.image.data.resize(static_cast<size_t>(r.width) * r.height * 3);
  check(tg_step_capture(s.handle(), indenter_velocity.data(), n_substeps, &r,
                        c.depth.values.data(), c.image.data.data()));
  return c;
}

// Batched control step over independent episodes (config 4): every state
// steps with its velocity and is captured, all submitted before any wait.
// Throws the first failing episode's error after all were processed.
inline std::vector<Capture> step_capture_many(std::vector<mpm::SimState*>& states,
                                              const std::vector<Vec3>& velocities,
                                              int n_substeps, const std::string& config_json,
                                              const std::string& object) {
  tg_render r;
  check(tg_render_from_config(config_json.c_str(), object.c_str(), &r));
  const size_t n = states.size();
  std::vector<Capture> out(n);
  std::vector<tg_handle> hs(n);
  std::vector<double> v(3 * n);
  std::vector<double*> dp(n);
  std::vector<uint8_t*> cp(n);
  for (size_t i = 0; i < n; ++i) {
    Capture& c = out[i];
    c.depth.width = c.image.width = r.width;
    c.depth.height = c.image.height = r.height;
    c.depth.pixel_to_meter = r.pixel_to_meter * r.crop_scale;
    c.depth.values.resize(static_cast<size_t>(r.width) * r.height);
    c.image.data.resize(static_cast<size_t>(r.width) * r.height * 3);
    hs[i] = states[i]->handle();
    for (int a = 0; a < 3; ++a) v[3 * i + a] = velocities[i][a];
    dp[i] = c.depth.values.data();
    cp[i] = c.image.data.data();
  }
  check(tg_step_capture_many(hs.data(), static_cast<int>(n), v.data(), n_substeps, &r, 1,
                             dp.data(), cp.data(), nullptr));
  return out;
}

}  // namespace sim

// ---- bridge (server.hpp:13-40), dataset (harness.hpp), metrics ------------
namespace bridge {
// run_protocol over newline-separated JSON messages; returns the reply lines.
inline std::string run_protocol(const std::string& input, const std::string& base_config_json,
                                const std::string& session_root, int device = 0) {
  char* out = nullptr;
  check(tg_bridge_run(device, base_config_json.c_str(), session_root.c_str(), input.c_str(), &out));
  std::string replies(out);
  tg_free(out);
  return replies;
}
// serve_stdio (port < 0) / serve_tcp on 127.0.0.1:port
inline void serve(const std::string& base_config_json, const std::string& session_root,
                  int port = -1, int max_connections = 0, int device = 0) {
  check(tg_bridge_serve(device, base_config_json.c_str(), session_root.c_str(), port,
                        max_connections));
}
}  // namespace bridge

namespace dataset {
struct DatasetResult {
  int64_t rows = 0, skipped_positions = 0;
};
inline DatasetResult run_press_dataset(const std::string& config_json, const std::string& out_dir,
                                       int device = 0, int batch = 0) {
  DatasetResult r;
  check(tg_run_press_dataset(device, config_json.c_str(), out_dir.c_str(), batch, &r.rows,
                             &r.skipped_positions));
  return r;
}
struct CompareAggregate {
  int64_t pairs = 0;
  double ssim_mean = 0, ssim_std = 0, psnr_mean = 0, psnr_std = 0, mae_mean = 0, mae_std = 0;
};
inline CompareAggregate compare_datasets(const std::string& dir_a, const std::string& dir_b,
                                         const std::string& csv_out = "", int device = 0) {
  double o[7];
  check(tg_compare_datasets(device, dir_a.c_str(), dir_b.c_str(), csv_out.c_str(), o));
  return {static_cast<int64_t>(o[0]), o[1], o[2], o[3], o[4], o[5], o[6]};
}
}  // namespace dataset

namespace metrics {
struct MetricReport {
  double ssim = 0, psnr_db = 0, mae_pct = 0;
};
inline MetricReport compare(const render::Image8& a, const render::Image8& b, int device = 0) {
  if (a.width != b.width || a.height != b.height)
    throw ShapeMismatch("image shapes differ");
  double o[3];
  check(tg_image_metrics(device, a.data.data(), b.data.data(), a.width, a.height, 1, o));
  return {o[0], o[1], o[2]};
}
}  // namespace metrics
}  // namespace tacchi_b200
