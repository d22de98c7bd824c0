// oracle/_ref driver — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper around the UNMODIFIED reference sources under
// /root/reference/proj (compiled by oracle/Makefile against the Eigen-subset
// shim in oracle/eigen_shim). It exists so that pytest (via ctypes) and
// bench.py's `--impl reference` / cpu_baseline leg can drive the reference's
// own C++ API: sim::build_sim (scene_builder.cpp:63-78), mpm::step and its six
// phases (engine.cpp:53-297), sim::capture (scene_builder.cpp:80-89), the
// render functions (depth_extract.cpp, depth_map.cpp, phong.cpp), the geometry
// generators (shapes.cpp, particle_set.cpp) and the serial test oracle
// tests/oracle/reference_mpm.cpp.
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
// legs may load the resulting library. The product never links it.
//
// Particle arrays cross this boundary in "row layout": x, v as N x 3; C, F as
// N x 9 with M(i,j) at [9p + 3i + j].
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <cstdio>
#include <cstdlib>
#include <sstream>

#include "oracle/reference_mpm.hpp"
#include "tacchi/bridge/server.hpp"
#include "tacchi/dataset/harness.hpp"
#include "tacchi/metrics/image_metrics.hpp"
#include "tacchi/config/scene_config.hpp"
#include "tacchi/errors.hpp"
#include "tacchi/geo/particle_set.hpp"
#include "tacchi/geo/shapes.hpp"
#include "tacchi/mpm/engine.hpp"
#include "tacchi/mpm/material.hpp"
#include "tacchi/mpm/sim_state.hpp"
#include "tacchi/render/depth_extract.hpp"
#include "tacchi/render/depth_map.hpp"
#include "tacchi/render/image.hpp"
#include "tacchi/render/phong.hpp"
#include "tacchi/sim/scene_builder.hpp"

using namespace tacchi;

// PNG I/O (render/image.cpp) needs libpng, which is absent here. The hot path
// never calls it; the bridge (session.cpp:47) does, so save_png is replaced by
// a writer of the same pixels in binary PPM ("P6 w h 255" + RGB rows) under
// the requested name — the bridge parity test decodes both formats and
// compares pixels.
namespace tacchi::render {
void save_png(const Image8& image, const std::filesystem::path& path) {
  if (image.width <= 0 || image.height <= 0) throw IoError("save_png: empty image");
  std::FILE* f = std::fopen(path.string().c_str(), "wb");
  if (!f) throw IoError("cannot write " + path.string());
  std::fprintf(f, "P6\n%d %d\n255\n", image.width, image.height);
  std::fwrite(image.data.data(), 1, image.data.size(), f);
  std::fclose(f);
}
// ... and load_png reads that PPM back (render_params_struct's background).
Image8 load_png(const std::filesystem::path& path) {
  std::FILE* f = std::fopen(path.string().c_str(), "rb");
  if (!f) throw IoError("cannot open " + path.string());
  int w = 0, h = 0, maxv = 0;
  if (std::fscanf(f, "P6 %d %d %d", &w, &h, &maxv) != 3 || maxv != 255 || w <= 0 || h <= 0) {
    std::fclose(f);
    throw ParseError("not a binary PPM (oracle build): " + path.string());
  }
  std::fgetc(f);  // the single whitespace after the header
  Image8 img(w, h);
  const size_t got = std::fread(img.data.data(), 1, img.data.size(), f);
  std::fclose(f);
  if (got != img.data.size()) throw ParseError("truncated PPM: " + path.string());
  return img;
}
}  // namespace tacchi::render

namespace {

thread_local std::string g_err;

// Error codes shared with include/tacchi_cuda.h (TG_ERR_*).
int code_of(const std::exception& e) {
  if (dynamic_cast<const GridTooSmall*>(&e)) return 1;
  if (dynamic_cast<const EmptyScene*>(&e)) return 2;
  if (dynamic_cast<const OutOfGrid*>(&e)) return 3;
  if (dynamic_cast<const DegenerateF*>(&e)) return 4;
  if (dynamic_cast<const ConfigError*>(&e)) return 5;
  if (dynamic_cast<const NoSurface*>(&e)) return 6;
  if (dynamic_cast<const CropOutOfBounds*>(&e)) return 7;
  if (dynamic_cast<const ShapeMismatch*>(&e)) return 8;
  if (dynamic_cast<const EmptyCloud*>(&e)) return 9;
  if (dynamic_cast<const ParseError*>(&e)) return 10;
  if (dynamic_cast<const IoError*>(&e)) return 11;
  if (dynamic_cast<const SessionNotInitialized*>(&e)) return 12;
  if (dynamic_cast<const NonMonotonicTime*>(&e)) return 13;
  if (dynamic_cast<const ProtocolError*>(&e)) return 14;
  if (dynamic_cast<const ManifestMismatch*>(&e)) return 15;
  return 99;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

struct RefSim {
  mpm::SimState state;
};

void put_vec(const Vec3& v, double* out) { out[0] = v.x(); out[1] = v.y(); out[2] = v.z(); }
void put_mat(const Mat3& m, double* out) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) out[3 * i + j] = m(i, j);
}
Mat3 get_mat(const double* in) {
  Mat3 m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m(i, j) = in[3 * i + j];
  return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Full reference scene setup: config JSON (partial overrides of default_config),
// indenter object name, lateral press offset (m). Mirrors the harness / session
// setup path: indenter_cloud_for -> place_for_press -> build_sim.
int ref_build(const char* cfg_json, const char* object, double off_x, double off_y,
              int num_threads, void** out) {
  return guard([&] {
    const config::SceneConfig cfg = config::from_json_string(cfg_json);
    const geo::ParticleSet cloud = sim::indenter_cloud_for(cfg, object ? object : "");
    const geo::ParticleSet placed = sim::place_for_press(cfg, cloud, off_x, off_y);
    auto* s = new RefSim{sim::build_sim(cfg, placed, num_threads)};
    *out = s;
  });
}

// Engine-level setup from explicit parts (tests): SceneParams fields, lattice
// (dims, counts, origin) and an indenter position list (N x 3, meters).
int ref_build_parts(const int res[3], double grid_edge, const double grid_origin[3],
                    double E, double nu, double rho, double dt, int fixed_bottom_layers,
                    const double gravity[3], double indenter_mass_scale,
                    const double lat_dims[3], const int lat_counts[3], const double lat_origin[3],
                    const double* ind_pos, long n_ind, const double ind_v0[3], int num_threads,
                    void** out) {
  return guard([&] {
    mpm::SceneParams p;
    p.grid_resolution = Vec3i(res[0], res[1], res[2]);
    p.grid_edge = grid_edge;
    p.grid_origin = Vec3(grid_origin[0], grid_origin[1], grid_origin[2]);
    p.material.youngs_modulus = E;
    p.material.poisson_ratio = nu;
    p.material.density = rho;
    p.dt = dt;
    p.fixed_bottom_layers = fixed_bottom_layers;
    p.gravity = Vec3(gravity[0], gravity[1], gravity[2]);
    p.indenter_mass_scale = indenter_mass_scale;
    const geo::ParticleSet el = geo::make_elastomer_lattice(
        Vec3(lat_dims[0], lat_dims[1], lat_dims[2]),
        Vec3i(lat_counts[0], lat_counts[1], lat_counts[2]),
        Vec3(lat_origin[0], lat_origin[1], lat_origin[2]));
    geo::ParticleSet ind;
    ind.tag = geo::Tag::Indenter;
    for (long i = 0; i < n_ind; ++i)
      ind.positions.emplace_back(ind_pos[3 * i], ind_pos[3 * i + 1], ind_pos[3 * i + 2]);
    auto* s = new RefSim{mpm::init_scene(p, el, ind, Vec3(ind_v0[0], ind_v0[1], ind_v0[2]))};
    s->state.num_threads = num_threads;
    *out = s;
  });
}

void ref_destroy(void* h) { delete static_cast<RefSim*>(h); }
long ref_num_particles(void* h) { return static_cast<long>(static_cast<RefSim*>(h)->state.particles.size()); }
long ref_elastomer_count(void* h) { return static_cast<long>(static_cast<RefSim*>(h)->state.elastomer_count); }
void ref_set_threads(void* h, int n) { static_cast<RefSim*>(h)->state.num_threads = n; }

int ref_get_state(void* h, double* x, double* v, double* C, double* F, double* mass,
                  double* vol0, uint8_t* tag) {
  return guard([&] {
    const auto& ps = static_cast<RefSim*>(h)->state.particles;
    for (std::size_t p = 0; p < ps.size(); ++p) {
      if (x) put_vec(ps.x[p], x + 3 * p);
      if (v) put_vec(ps.v[p], v + 3 * p);
      if (C) put_mat(ps.C[p], C + 9 * p);
      if (F) put_mat(ps.F[p], F + 9 * p);
      if (mass) mass[p] = ps.mass[p];
      if (vol0) vol0[p] = ps.volume0[p];
      if (tag) tag[p] = static_cast<uint8_t>(ps.tag[p]);
    }
  });
}

int ref_set_state(void* h, const double* x, const double* v, const double* C, const double* F) {
  return guard([&] {
    auto& ps = static_cast<RefSim*>(h)->state.particles;
    for (std::size_t p = 0; p < ps.size(); ++p) {
      if (x) ps.x[p] = Vec3(x[3 * p], x[3 * p + 1], x[3 * p + 2]);
      if (v) ps.v[p] = Vec3(v[3 * p], v[3 * p + 1], v[3 * p + 2]);
      if (C) ps.C[p] = get_mat(C + 9 * p);
      if (F) ps.F[p] = get_mat(F + 9 * p);
    }
  });
}

int ref_step(void* h, const double vind[3], int n_substeps) {
  return guard([&] {
    mpm::step(static_cast<RefSim*>(h)->state, Vec3(vind[0], vind[1], vind[2]), n_substeps);
  });
}

// phase: 0 zero_grid, 1 particle_to_grid, 2 grid_update, 3 grid_to_particle,
// 4 apply_boundary(v), 5 advect.
int ref_phase(void* h, int phase, const double vind[3]) {
  return guard([&] {
    auto& st = static_cast<RefSim*>(h)->state;
    switch (phase) {
      case 0: mpm::zero_grid(st); break;
      case 1: mpm::particle_to_grid(st); break;
      case 2: mpm::grid_update(st); break;
      case 3: mpm::grid_to_particle(st); break;
      case 4: mpm::apply_boundary(st, Vec3(vind[0], vind[1], vind[2])); break;
      case 5: mpm::advect(st); break;
      default: throw ConfigError("bad phase id");
    }
  });
}

void ref_get_diag(void* h, double* min_det_f, double* max_speed, long* step_count,
                  double* indenter_velocity) {
  const auto& st = static_cast<RefSim*>(h)->state;
  *min_det_f = st.diag.min_det_f;
  *max_speed = st.diag.max_speed;
  *step_count = static_cast<long>(st.step_count);
  if (indenter_velocity) put_vec(st.indenter_velocity, indenter_velocity);
}

void ref_grid_info(void* h, int res[3], double* dx, double origin[3], int lo[3], int hi[3]) {
  const auto& g = static_cast<RefSim*>(h)->state.grid;
  for (int a = 0; a < 3; ++a) {
    res[a] = g.res[a];
    origin[a] = g.origin[a];
    lo[a] = g.active_lo[a];
    hi[a] = g.active_hi[a];
  }
  *dx = g.dx;
}

// Copies the node box [lo, hi) (k fastest) of mass / momentum / velocity.
int ref_get_grid(void* h, const int lo[3], const int hi[3], double* mass, double* mom,
                 double* vel) {
  return guard([&] {
    const auto& g = static_cast<RefSim*>(h)->state.grid;
    std::size_t o = 0;
    for (int i = lo[0]; i < hi[0]; ++i)
      for (int j = lo[1]; j < hi[1]; ++j)
        for (int k = lo[2]; k < hi[2]; ++k, ++o) {
          const std::size_t n = g.index(i, j, k);
          if (mass) mass[o] = g.mass[n];
          if (mom) put_vec(g.momentum[n], mom + 3 * o);
          if (vel) put_vec(g.velocity[n], vel + 3 * o);
        }
  });
}

void ref_surface(void* h, int* nx, int* ny, double geom[5], uint32_t* idx) {
  const auto& s = static_cast<RefSim*>(h)->state.surface;
  *nx = s.nx;
  *ny = s.ny;
  geom[0] = s.x0; geom[1] = s.y0; geom[2] = s.sx; geom[3] = s.sy; geom[4] = s.z0;
  if (idx) std::memcpy(idx, s.particle.data(), s.particle.size() * sizeof(uint32_t));
}

// sim::capture with the given config (lights/render/alignment) and object name.
int ref_capture(void* h, const char* cfg_json, const char* object, double* depth, uint8_t* rgb,
                int* out_w, int* out_h) {
  return guard([&] {
    const config::SceneConfig cfg = config::from_json_string(cfg_json);
    const sim::Capture cap = sim::capture(static_cast<RefSim*>(h)->state, cfg, object ? object : "");
    *out_w = cap.depth.width;
    *out_h = cap.depth.height;
    if (depth) std::memcpy(depth, cap.depth.values.data(), cap.depth.values.size() * sizeof(double));
    if (rgb) std::memcpy(rgb, cap.image.data.data(), cap.image.data.size());
  });
}

// extract_surface_depth; w or h <= 0 selects the full-surface overload.
int ref_extract_depth(void* h, int w, int hgt, double r, double* out, int* out_w, int* out_h) {
  return guard([&] {
    const auto& st = static_cast<RefSim*>(h)->state;
    const render::DepthMap m = (w > 0 && hgt > 0) ? render::extract_surface_depth(st, w, hgt, r)
                                                  : render::extract_surface_depth(st, r);
    *out_w = m.width;
    *out_h = m.height;
    if (out) std::memcpy(out, m.values.data(), m.values.size() * sizeof(double));
  });
}

int ref_crop_align(const double* src, int sw, int sh, double r, double off_x, double off_y,
                   double scale, int ow, int oh, double* out, double* out_r) {
  return guard([&] {
    render::DepthMap m;
    m.width = sw;
    m.height = sh;
    m.pixel_to_meter = r;
    m.values.assign(src, src + static_cast<std::size_t>(sw) * sh);
    render::CropAlignment a;
    a.offset_x = off_x;
    a.offset_y = off_y;
    a.scale = scale;
    const render::DepthMap o = render::crop_align(m, a, ow, oh);
    std::memcpy(out, o.values.data(), o.values.size() * sizeof(double));
    if (out_r) *out_r = o.pixel_to_meter;
  });
}

int ref_surface_normals(const double* d, int w, int hgt, double r, double* out) {
  return guard([&] {
    render::DepthMap m;
    m.width = w;
    m.height = hgt;
    m.pixel_to_meter = r;
    m.values.assign(d, d + static_cast<std::size_t>(w) * hgt);
    const render::NormalMap nm = render::surface_normals(m);
    for (std::size_t i = 0; i < nm.normals.size(); ++i) put_vec(nm.normals[i], out + 3 * i);
  });
}

// phong_render with the lights and RenderParams of the given config JSON.
int ref_phong(const double* d, int w, int hgt, double r, const char* cfg_json, uint8_t* out) {
  return guard([&] {
    const config::SceneConfig cfg = config::from_json_string(cfg_json);
    render::DepthMap m;
    m.width = w;
    m.height = hgt;
    m.pixel_to_meter = r;
    m.values.assign(d, d + static_cast<std::size_t>(w) * hgt);
    const render::Image8 img = render::phong_render(m, cfg.lights, cfg.render_params_struct());
    std::memcpy(out, img.data.data(), img.data.size());
  });
}

// Resolved lights (N x 9: direction, diffuse, specular) of a config JSON.
int ref_config_lights(const char* cfg_json, double* out, int* n) {
  return guard([&] {
    const config::SceneConfig cfg = config::from_json_string(cfg_json);
    *n = static_cast<int>(cfg.lights.size());
    if (out)
      for (std::size_t i = 0; i < cfg.lights.size(); ++i) {
        put_vec(cfg.lights[i].direction, out + 9 * i);
        put_vec(cfg.lights[i].diffuse, out + 9 * i + 3);
        put_vec(cfg.lights[i].specular, out + 9 * i + 6);
      }
  });
}

int ref_generate_cloud(const char* shape, long n, uint64_t seed, double* out) {
  return guard([&] {
    const geo::ParticleSet s = geo::generate_shape_cloud(shape, static_cast<std::size_t>(n), seed);
    for (std::size_t i = 0; i < s.size(); ++i) put_vec(s.positions[i], out + 3 * i);
  });
}

// indenter_cloud_for + place_for_press for a config; returns the count first
// when out == nullptr.
int ref_placed_indenter(const char* cfg_json, const char* object, double off_x, double off_y,
                        double* out, long* n) {
  return guard([&] {
    const config::SceneConfig cfg = config::from_json_string(cfg_json);
    const geo::ParticleSet cloud = sim::indenter_cloud_for(cfg, object ? object : "");
    const geo::ParticleSet placed = sim::place_for_press(cfg, cloud, off_x, off_y);
    *n = static_cast<long>(placed.size());
    if (out)
      for (std::size_t i = 0; i < placed.size(); ++i) put_vec(placed.positions[i], out + 3 * i);
  });
}

int ref_polar_rotation(const double* F, double* R) {
  return guard([&] { put_mat(mpm::polar_rotation(get_mat(F)), R); });
}
int ref_polar_rotation_svd(const double* F, double* R) {
  return guard([&] { put_mat(mpm::polar_rotation_svd(get_mat(F)), R); });
}
int ref_corotated_stress(const double* F, double E, double nu, double rho, double* S) {
  return guard([&] {
    mpm::MaterialParams m;
    m.youngs_modulus = E;
    m.poisson_ratio = nu;
    m.density = rho;
    put_mat(mpm::corotated_stress(get_mat(F), m), S);
  });
}

// tests/oracle/reference_mpm.cpp:reference_step on an explicit scene.
// State arrays are updated in place; the filled grid (nx*ny*nz nodes) is
// written to grid_mass / grid_mom / grid_vel when non-null.
int ref_oracle_step(long n, double* x, double* v, double* C, double* F, const double* mass,
                    const double* vol0, const uint8_t* tag, int nx, int ny, int nz, double dx,
                    const double origin[3], double mu, double lambda, double dt,
                    const double vind[3], double* grid_mass, double* grid_mom, double* grid_vel) {
  return guard([&] {
    test_oracle::RefScene sc;
    sc.nx = nx; sc.ny = ny; sc.nz = nz;
    sc.dx = dx;
    sc.origin = Vec3(origin[0], origin[1], origin[2]);
    sc.mu = mu;
    sc.lambda = lambda;
    sc.dt = dt;
    sc.particles.resize(static_cast<std::size_t>(n));
    for (long p = 0; p < n; ++p) {
      auto& q = sc.particles[p];
      q.x = Vec3(x[3 * p], x[3 * p + 1], x[3 * p + 2]);
      q.v = Vec3(v[3 * p], v[3 * p + 1], v[3 * p + 2]);
      q.C = get_mat(C + 9 * p);
      q.F = get_mat(F + 9 * p);
      q.mass = mass[p];
      q.volume0 = vol0[p];
      q.tag = tag[p];
    }
    const test_oracle::RefGrid g = test_oracle::reference_step(sc, Vec3(vind[0], vind[1], vind[2]));
    for (long p = 0; p < n; ++p) {
      const auto& q = sc.particles[p];
      put_vec(q.x, x + 3 * p);
      put_vec(q.v, v + 3 * p);
      put_mat(q.C, C + 9 * p);
      put_mat(q.F, F + 9 * p);
    }
    for (std::size_t i = 0; i < g.mass.size(); ++i) {
      if (grid_mass) grid_mass[i] = g.mass[i];
      if (grid_mom) put_vec(g.momentum[i], grid_mom + 3 * i);
      if (grid_vel) put_vec(g.velocity[i], grid_vel + 3 * i);
    }
  });
}

}  // extern "C"

// bridge::run_protocol (server.cpp:49-113) over in-memory lines, with the
// SceneConfig base parsed from `base_json`; replies returned malloc'd in *out.
extern "C" int ref_bridge_run(const char* base_json, const char* session_root, const char* input,
                              char** out) {
  return guard([&] {
    const config::SceneConfig base = config::from_json_string(base_json ? base_json : "{}");
    std::istringstream in(input ? input : "");
    std::string replies;
    bridge::run_protocol(
        [&in](std::string& l) { return static_cast<bool>(std::getline(in, l)); },
        [&replies](const std::string& l) {
          replies += l;
          replies += '\n';
        },
        base, session_root ? session_root : ".");
    *out = static_cast<char*>(std::malloc(replies.size() + 1));
    std::memcpy(*out, replies.c_str(), replies.size() + 1);
  });
}

extern "C" void ref_free(void* p) { std::free(p); }

// dataset::run_press_dataset (harness.cpp:159-245); images land as PPM under
// their .png names (save_png above).
extern "C" int ref_run_press_dataset(const char* cfg_json, const char* out_dir, long* rows,
                                     long* skipped) {
  return guard([&] {
    const config::SceneConfig cfg = config::from_json_string(cfg_json ? cfg_json : "{}");
    const dataset::DatasetResult r = dataset::run_press_dataset(cfg, out_dir);
    *rows = static_cast<long>(r.rows);
    *skipped = static_cast<long>(r.skipped_positions);
  });
}

// metrics::compare (image_metrics.cpp:110-112) on two h x w x 3 images.
extern "C" int ref_image_metrics(const uint8_t* a, const uint8_t* b, int w, int h, double* out) {
  return guard([&] {
    render::Image8 ia(w, h), ib(w, h);
    std::memcpy(ia.data.data(), a, static_cast<size_t>(w) * h * 3);
    std::memcpy(ib.data.data(), b, static_cast<size_t>(w) * h * 3);
    const metrics::MetricReport m = metrics::compare(ia, ib);
    out[0] = m.ssim;
    out[1] = m.psnr_db;
    out[2] = m.mae_pct;
  });
}
