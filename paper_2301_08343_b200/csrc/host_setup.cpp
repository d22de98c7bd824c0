// Host-side scene setup for the B200 path: SceneConfig JSON, the indenter
// geometry generators and sim::build_sim / sim::capture's parameter
// resolution. This is once-per-episode host work (SURVEY §2.1 "Geometry",
// "Config"); it must reproduce the reference's inputs bit-for-bit so that the
// device hot path sees identical particles. References are to
// /root/reference/proj.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <charconv>
#include <filesystem>
#include <fstream>
#include <string_view>
#include <functional>
#include <memory>
#include <mutex>
#include <map>
#include <numeric>
#include <random>
#include <string>
#include <vector>
#include <thread>
#include <atomic>

#include <nlohmann/json.hpp>

#include "tacchi_cuda.h"

#include "host_config.hpp"
#include "setup_shapes.h"

namespace tacchi_b200 {
int fail(int code, const std::string& msg);
}

namespace tacchi_b200::host {

using tacchi_b200::fail;
using json = nlohmann::json;

// scene_config.cpp:42-57: three tinted lights, 120 deg apart, 45 deg elevation.
std::vector<Light> default_rig() {
  std::vector<Light> rig;
  const double e = std::sqrt(0.5);
  const double tints[3][3] = {{0.80, 0.12, 0.10}, {0.10, 0.80, 0.12}, {0.12, 0.10, 0.80}};
  for (int m = 0; m < 3; ++m) {
    const double az = 2.0 * M_PI * m / 3.0;
    Light l;
    l.dir[0] = e * std::cos(az);
    l.dir[1] = e * std::sin(az);
    l.dir[2] = -e;
    for (int c = 0; c < 3; ++c) {
      l.diffuse[c] = tints[m][c];
      l.specular[c] = 0.5 * tints[m][c];
    }
    rig.push_back(l);
  }
  return rig;
}

void read3(const json& j, const char* key, double* out) {
  if (!j.contains(key)) return;
  const json& a = j.at(key);
  if (!a.is_array() || a.size() != 3) raise(TG_ERR_CONFIG, "expected a 3-element array");
  for (int i = 0; i < 3; ++i) out[i] = a[i].get<double>();
}
void read3i(const json& j, const char* key, int* out) {
  if (!j.contains(key)) return;
  const json& a = j.at(key);
  if (!a.is_array() || a.size() != 3) raise(TG_ERR_CONFIG, "expected a 3-element array");
  for (int i = 0; i < 3; ++i) out[i] = a[i].get<int>();
}
template <typename T>
void read(const json& j, const char* key, T& out) {
  if (j.contains(key)) out = j.at(key).get<T>();
}

void normalize(double* v) {  // Eigen normalized(): v / sqrt(squaredNorm) if > 0
  const double n2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  if (n2 > 0.0) {
    const double n = std::sqrt(n2);
    v[0] /= n; v[1] /= n; v[2] /= n;
  }
}

[[noreturn]] void raise(int code, const std::string& msg) { throw HostError{code, msg}; }

// from_json_string (scene_config.cpp:187-257): partial overrides of defaults.
Config parse_config(const char* text) {
  Config c;
  c.lights = default_rig();
  if (!text || !*text) return c;
  json j = json::parse(text, nullptr, false);
  if (j.is_discarded()) raise(TG_ERR_CONFIG, "config is not valid JSON");
  try {
    if (j.contains("elastomer")) {
      const json& e = j["elastomer"];
      read3(e, "size_mm", c.size_mm);
      read3i(e, "particle_counts", c.counts);
      read(e, "youngs_modulus_pa", c.E);
      read(e, "poisson_ratio", c.nu);
      read(e, "density_kg_m3", c.rho);
      read(e, "fixed_bottom_layers", c.fixed_bottom_layers);
    }
    if (j.contains("grid")) {
      read3i(j["grid"], "nodes_per_axis", c.nodes);
      read(j["grid"], "edge_mm", c.edge_mm);
    }
    if (j.contains("time")) {
      read(j["time"], "dt_s", c.dt);
      read(j["time"], "substeps_per_control_step", c.substeps_per_control_step);
      read(j["time"], "press_speed_mm_s", c.press_speed_mm_s);
    }
    if (j.contains("indenter")) {
      const json& i = j["indenter"];
      read(i, "cloud_path", c.cloud_path);
      read(i, "generated_shape", c.generated_shape);
      read(i, "source_points", c.source_points);
      read(i, "target_points", c.target_points);
      read(i, "seed", c.seed);
      read(i, "gap_mm", c.gap_mm);
      read(i, "z_rotation_rad", c.z_rotation_rad);
      read(i, "rigid_mass_scale", c.rigid_mass_scale);
    }
    if (j.contains("lights")) {
      c.lights.clear();
      for (const json& lj : j["lights"]) {
        Light l{{0, 0, -1}, {1, 1, 1}, {0, 0, 0}};
        if (!lj.contains("direction")) raise(TG_ERR_CONFIG, "light without direction");
        read3(lj, "direction", l.dir);
        normalize(l.dir);  // scene_config.cpp:220
        read3(lj, "diffuse_rgb", l.diffuse);
        read3(lj, "specular_rgb", l.specular);
        c.lights.push_back(l);
      }
    }
    if (j.contains("render")) {
      const json& r = j["render"];
      read(r, "ambient_k", c.ka);
      read(r, "diffuse_k", c.kd);
      read(r, "specular_k", c.ks);
      read(r, "shininess", c.shininess);
      read3(r, "ambient_rgb", c.ambient);
      read3(r, "view_dir", c.view);
      read(r, "pixel_to_meter", c.pixel_to_meter);
      read(r, "image_width", c.image_w);
      read(r, "image_height", c.image_h);
      read(r, "background_image", c.background_image);
    }
    if (j.contains("alignment")) {
      for (auto it = j["alignment"].begin(); it != j["alignment"].end(); ++it) {
        Config::Align a;
        const json& aj = it.value();
        if (aj.contains("offset_px")) {
          a.ox = aj["offset_px"][0].get<double>();
          a.oy = aj["offset_px"][1].get<double>();
        }
        read(aj, "scale", a.scale);
        c.alignment[it.key()] = a;
      }
    }
    if (j.contains("press_grid")) {
      const json& p = j["press_grid"];
      read(p, "positions_x", c.positions_x);
      read(p, "positions_y", c.positions_y);
      read(p, "step_mm", c.step_mm);
      if (p.contains("depths_mm")) c.depths_mm = p["depths_mm"].get<std::vector<double>>();
    }
    if (j.contains("objects")) c.objects = j["objects"].get<std::vector<std::string>>();
    read(j, "output_dir", c.output_dir);
    read(j, "deterministic", c.deterministic);
    read(j, "workers", c.workers);
    read(j, "gravity_mps2", c.gravity_mps2);
  } catch (const json::exception& e) {
    raise(TG_ERR_CONFIG, std::string("config: ") + e.what());
  }
  return c;
}

// ---- geometry (geo/shapes.cpp, geo/particle_set.cpp) ----------------------

constexpr double kPi = 3.14159265358979323846;

double sq(double v) { return v * v; }
double r2(double x, double y) { return x * x + y * y; }
bool disk(double x, double y, double r) { return r2(x, y) <= r * r; }
bool rect(double x, double y, double hx, double hy) { return std::abs(x) <= hx && std::abs(y) <= hy; }

// Half-plane tests of a regular polygon / equilateral triangle (shapes.cpp:33-52).
bool polygon(double x, double y, int sides, double circumradius) {
  const double apothem = circumradius * std::cos(kPi / sides);
  for (int k = 0; k < sides; ++k) {
    const double a = (2.0 * kPi * k + kPi) / sides;
    if (x * std::cos(a) + y * std::sin(a) > apothem) return false;
  }
  return true;
}
bool triangle(double x, double y, double side) {
  const double r = side / std::sqrt(3.0);
  const double apothem = r / 2.0;
  for (int k = 0; k < 3; ++k) {
    const double a = -kPi / 2.0 + 2.0 * kPi * k / 3.0;
    if (x * std::cos(a) + y * std::sin(a) > apothem) return false;
  }
  return true;
}

// The "random" shape's fixed bump field (shapes.cpp:56-77).
struct Bumps {
  double cx[28], cy[28], amp[28], inv_s2[28];
  Bumps() {
    std::mt19937_64 rng(0x7ac371u);
    auto u = [&rng]() { return (rng() >> 11) * 0x1.0p-53; };
    for (int i = 0; i < 28; ++i) {
      cx[i] = -3.2 + 6.4 * u();
      cy[i] = -3.2 + 6.4 * u();
      amp[i] = 0.25 + 0.85 * u();
      const double s = 0.45 + 0.75 * u();
      inv_s2[i] = 1.0 / (2.0 * s * s);
    }
  }
  double height(double x, double y) const {
    double h = 0.0;
    for (int i = 0; i < 28; ++i) h += amp[i] * std::exp(-(sq(x - cx[i]) + sq(y - cy[i])) * inv_s2[i]);
    return std::min(h, 1.4);
  }
};

struct Shape {
  double lo[3], hi[3];  // mm
  std::function<bool(double, double, double)> inside;
};

// The 21 analytic indenter solids (shapes.cpp:79-206), millimetres, contact
// feature facing -z with the lowest material at z = 0.
bool make_shape(const std::string& name, Shape& s) {
  auto box = [&](double x0, double y0, double z0, double x1, double y1, double z1) {
    s.lo[0] = x0; s.lo[1] = y0; s.lo[2] = z0;
    s.hi[0] = x1; s.hi[1] = y1; s.hi[2] = z1;
  };
  if (name == "sphere") {
    box(-3, -3, 0, 3, 3, 6);
    s.inside = [](double x, double y, double z) { return r2(x, y) + sq(z - 3.0) <= 9.0; };
  } else if (name == "sphere2") {
    box(-2, -2, 0, 2, 2, 4);
    s.inside = [](double x, double y, double z) { return r2(x, y) + sq(z - 2.0) <= 4.0; };
  } else if (name == "cone") {
    box(-3.5, -3.5, 0, 3.5, 3.5, 3.5);
    s.inside = [](double x, double y, double z) { return r2(x, y) <= z * z && z <= 3.5; };
  } else if (name == "cylinder") {
    box(-3, -3, 0, 3, 3, 3);
    s.inside = [](double x, double y, double) { return disk(x, y, 3.0); };
  } else if (name == "cylinder_shell") {
    box(-3, -3, 0, 3, 3, 3);
    s.inside = [](double x, double y, double) {
      const double q = r2(x, y);
      return q <= 9.0 && q >= sq(2.1);
    };
  } else if (name == "cylinder_side") {
    box(-2, -4, 0, 2, 4, 4);
    s.inside = [](double x, double, double z) { return sq(x) + sq(z - 2.0) <= 4.0; };
  } else if (name == "curved_surface") {
    box(-4, -4, 0, 4, 4, 3);
    s.inside = [](double x, double y, double z) { return z >= r2(x, y) / 24.0; };
  } else if (name == "flat_slab") {
    box(-4, -4, 0, 4, 4, 3);
    s.inside = [](double, double, double) { return true; };
  } else if (name == "dot_in") {
    box(-3.5, -3.5, 0, 3.5, 3.5, 3);
    s.inside = [](double x, double y, double z) {
      return disk(x, y, 3.5) && !(disk(x, y, 0.7) && z < 0.9);
    };
  } else if (name == "dots") {
    box(-3.5, -3.5, 0, 3.5, 3.5, 3);
    s.inside = [](double x, double y, double z) {
      if (z >= 1.0) return rect(x, y, 3.5, 3.5);
      const double gx = std::round(x / 2.2) * 2.2;
      const double gy = std::round(y / 2.2) * 2.2;
      return std::abs(gx) <= 2.3 && std::abs(gy) <= 2.3 && disk(x - gx, y - gy, 0.55);
    };
  } else if (name == "hexagon") {
    box(-3.5, -3.5, 0, 3.5, 3.5, 3);
    s.inside = [](double x, double y, double) { return polygon(x, y, 6, 3.5); };
  } else if (name == "triangle") {
    box(-4, -4, 0, 4, 4, 3);
    s.inside = [](double x, double y, double) { return triangle(x, y, 6.5); };
  } else if (name == "prism") {
    box(-3, -4, 0, 3, 4, 3);
    s.inside = [](double x, double, double z) { return std::abs(x) <= z && z <= 3.0; };
  } else if (name == "line") {
    box(-0.6, -4, 0, 0.6, 4, 2);
    s.inside = [](double x, double y, double) { return rect(x, y, 0.6, 4.0); };
  } else if (name == "parallel_lines") {
    box(-3.4, -4, 0, 3.4, 4, 3);
    s.inside = [](double x, double y, double z) {
      if (z >= 1.5) return rect(x, y, 3.4, 4.0);
      const double gx = std::round(x / 2.4) * 2.4;
      return std::abs(gx) <= 2.5 && std::abs(x - gx) <= 0.45 && std::abs(y) <= 4.0;
    };
  } else if (name == "cross_lines") {
    box(-4, -4, 0, 4, 4, 3);
    s.inside = [](double x, double y, double z) {
      if (z >= 1.5) return rect(x, y, 4.0, 4.0);
      return (std::abs(x) <= 0.45 || std::abs(y) <= 0.45) && rect(x, y, 4.0, 4.0);
    };
  } else if (name == "moon") {
    box(-3, -3, 0, 3, 3, 2);
    s.inside = [](double x, double y, double) { return disk(x, y, 3.0) && !disk(x - 1.4, y, 2.4); };
  } else if (name == "pacman") {
    box(-3, -3, 0, 3, 3, 2);
    s.inside = [](double x, double y, double) {
      return disk(x, y, 3.0) && std::abs(std::atan2(y, x)) > kPi / 6.0;
    };
  } else if (name == "torus") {
    box(-3.2, -3.2, 0, 3.2, 3.2, 1.8);
    s.inside = [](double x, double y, double z) {
      const double rho = std::sqrt(r2(x, y));
      return sq(rho - 2.3) + sq(z - 0.9) <= sq(0.9);
    };
  } else if (name == "wave1") {
    box(-4, -4, 0, 4, 4, 3);
    s.inside = [](double x, double, double z) {
      return z >= 0.5 * (1.0 + std::sin(2.0 * kPi * x / 2.7));
    };
  } else if (name == "random") {
    static const Bumps field;
    box(-4, -4, 0, 4, 4, 3);
    s.inside = [](double x, double y, double z) { return z >= field.height(x, y); };
  } else {
    return false;
  }
  return true;
}

// The device sampler's view of a shape (setup_shapes.h): its box and the
// libm constants of its predicate, evaluated here exactly as the host
// predicates above evaluate them.
bool shape_table(const std::string& name, ShapeTable& t) {
  static const char* kNames[] = {"sphere", "sphere2", "cone", "cylinder", "cylinder_shell",
                                 "cylinder_side", "curved_surface", "flat_slab", "dot_in", "dots",
                                 "hexagon", "triangle", "prism", "line", "parallel_lines",
                                 "cross_lines", "moon", "pacman", "torus", "wave1", "random"};
  Shape sh;
  if (!make_shape(name, sh)) return false;
  std::memset(&t, 0, sizeof(t));
  t.id = -1;
  for (int i = 0; i < 21; ++i)
    if (name == kNames[i]) t.id = i;
  if (t.id < 0) return false;
  for (int a = 0; a < 3; ++a) {
    t.lo[a] = sh.lo[a];
    t.span[a] = sh.hi[a] - sh.lo[a];
  }
  if (t.id == kShHexagon) {  // polygon(x, y, 6, 3.5)
    t.n_planes = 6;
    t.apothem = 3.5 * std::cos(kPi / 6);
    for (int k = 0; k < 6; ++k) {
      const double a = (2.0 * kPi * k + kPi) / 6;
      t.ca[k] = std::cos(a);
      t.sa[k] = std::sin(a);
    }
  } else if (t.id == kShTriangle) {  // triangle(x, y, 6.5)
    t.n_planes = 3;
    const double r = 6.5 / std::sqrt(3.0);
    t.apothem = r / 2.0;
    for (int k = 0; k < 3; ++k) {
      const double a = -kPi / 2.0 + 2.0 * kPi * k / 3.0;
      t.ca[k] = std::cos(a);
      t.sa[k] = std::sin(a);
    }
  } else if (t.id == kShRandom) {
    static const Bumps field;
    for (int i = 0; i < 28; ++i) {
      t.bx[i] = field.cx[i];
      t.by[i] = field.cy[i];
      t.amp[i] = field.amp[i];
      t.inv_s2[i] = field.inv_s2[i];
    }
  }
  return true;
}

bool is_known_shape(const std::string& name) {
  Shape s;
  return make_shape(name, s);
}

// generate_shape_cloud (shapes.cpp:231-249): rejection sampling, mm -> m.
std::vector<V3> generate_cloud(const std::string& name, size_t n, uint64_t seed) {
  Shape s;
  if (!make_shape(name, s)) raise(TG_ERR_CONFIG, "unknown shape: " + name);
  std::mt19937_64 rng(seed);
  auto u = [&rng]() { return (rng() >> 11) * 0x1.0p-53; };
  const double span[3] = {s.hi[0] - s.lo[0], s.hi[1] - s.lo[1], s.hi[2] - s.lo[2]};
  std::vector<V3> out;
  out.reserve(n);
  while (out.size() < n) {
    const double x = s.lo[0] + span[0] * u();
    const double y = s.lo[1] + span[1] * u();
    const double z = s.lo[2] + span[2] * u();
    if (s.inside(x, y, z)) out.push_back({x * 1e-3, y * 1e-3, z * 1e-3});
  }
  return out;
}

// Bounded draw by rejection (particle_set.cpp:48-56).
uint64_t draw_below(std::mt19937_64& rng, uint64_t bound) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t x;
  do {
    x = rng();
  } while (x >= limit);
  return x % bound;
}

// subsample (particle_set.cpp:60-90): partial Fisher-Yates, order-preserving.
std::vector<V3> subsample(const std::vector<V3>& cloud, size_t target, uint64_t seed) {
  if (target < 1) target = 1;
  const size_t n = cloud.size();
  if (n == 0) raise(TG_ERR_EMPTY_CLOUD, "subsample: empty cloud");
  if (target >= n) return cloud;
  std::vector<uint32_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0u);
  std::mt19937_64 rng(seed);
  for (size_t i = 0; i < target; ++i) {
    const size_t j = i + static_cast<size_t>(draw_below(rng, n - i));
    std::swap(idx[i], idx[j]);
  }
  idx.resize(target);
  std::sort(idx.begin(), idx.end());
  std::vector<V3> out;
  out.reserve(target);
  for (uint32_t i : idx) out.push_back(cloud[i]);
  return out;
}

void bbox(const std::vector<V3>& pts, V3& lo, V3& hi) {
  if (pts.empty()) raise(TG_ERR_EMPTY_CLOUD, "bounding_box: empty particle set");
  lo = hi = pts.front();
  for (const V3& p : pts) {
    lo.x = std::min(lo.x, p.x); lo.y = std::min(lo.y, p.y); lo.z = std::min(lo.z, p.z);
    hi.x = std::max(hi.x, p.x); hi.y = std::max(hi.y, p.y); hi.z = std::max(hi.z, p.z);
  }
}

// place_indenter (particle_set.cpp:92-102): rotate about z, then translate.
std::vector<V3> place(const std::vector<V3>& cloud, const V3& t, double rot) {
  const double c = std::cos(rot), s = std::sin(rot);
  std::vector<V3> out(cloud.size());
  for (size_t i = 0; i < cloud.size(); ++i) {
    const V3& p = cloud[i];
    const double x = c * p.x - s * p.y;
    const double y = s * p.x + c * p.y;
    out[i] = {x + t.x, y + t.y, p.z + t.z};
  }
  return out;
}

// ---- point-cloud files (geo/point_cloud_io.cpp:14-141): plain XYZ or ASCII
// PLY, coordinates in millimetres -----------------------------------------
namespace {

std::vector<std::string_view> split_ws(std::string_view line) {
  std::vector<std::string_view> toks;
  size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && (line[i] == ' ' || line[i] == '\t' || line[i] == '\r')) ++i;
    size_t j = i;
    while (j < line.size() && line[j] != ' ' && line[j] != '\t' && line[j] != '\r') ++j;
    if (j > i) toks.push_back(line.substr(i, j - i));
    i = j;
  }
  return toks;
}

bool parse_double(std::string_view tok, double& out) {
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), out);
  return r.ec == std::errc{} && r.ptr == tok.data() + tok.size();
}

bool parse_size(std::string_view tok, size_t& out) {
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), out);
  return r.ec == std::errc{} && r.ptr == tok.data() + tok.size();
}

[[noreturn]] void cloud_fail(const std::string& path, size_t line_no, const std::string& what) {
  raise(TG_ERR_PARSE, path + ":" + std::to_string(line_no) + ": " + what);
}

constexpr double kFileUnitToMeter = 1e-3;

std::vector<V3> load_ply(std::ifstream& in, const std::string& path) {
  std::string line;
  size_t line_no = 1;
  bool ascii = false, in_vertex = false;
  size_t vertex_count = 0;
  int xi = -1, yi = -1, zi = -1, props = 0;
  while (std::getline(in, line)) {
    ++line_no;
    const auto t = split_ws(line);
    if (t.empty() || t[0] == "comment") continue;
    if (t[0] == "format") {
      if (t.size() < 2 || t[1] != "ascii") cloud_fail(path, line_no, "only ascii PLY is supported");
      ascii = true;
    } else if (t[0] == "element") {
      if (t.size() < 3) cloud_fail(path, line_no, "malformed element line");
      in_vertex = t[1] == "vertex";
      if (in_vertex && !parse_size(t[2], vertex_count)) cloud_fail(path, line_no, "bad vertex count");
    } else if (t[0] == "property") {
      if (!in_vertex) continue;
      if (t.size() >= 3 && t[1] == "list") cloud_fail(path, line_no, "list property in vertex element");
      const std::string_view name = t.back();
      if (name == "x") xi = props;
      else if (name == "y") yi = props;
      else if (name == "z") zi = props;
      ++props;
    } else if (t[0] == "end_header") {
      break;
    }
  }
  if (!ascii) cloud_fail(path, line_no, "missing 'format ascii 1.0' header");
  if (xi < 0 || yi < 0 || zi < 0) cloud_fail(path, line_no, "vertex element lacks x/y/z properties");
  std::vector<V3> pts;
  pts.reserve(vertex_count);
  for (size_t v = 0; v < vertex_count; ++v) {
    if (!std::getline(in, line)) cloud_fail(path, line_no, "unexpected end of file in vertex data");
    ++line_no;
    const auto t = split_ws(line);
    if (t.empty()) {
      --v;
      continue;
    }
    if (static_cast<int>(t.size()) < props) cloud_fail(path, line_no, "short vertex line");
    double c[3];
    for (int a = 0; a < 3; ++a)
      if (!parse_double(t[a == 0 ? xi : (a == 1 ? yi : zi)], c[a]))
        cloud_fail(path, line_no, "bad coordinate");
    pts.push_back({c[0] * kFileUnitToMeter, c[1] * kFileUnitToMeter, c[2] * kFileUnitToMeter});
  }
  if (pts.empty()) raise(TG_ERR_EMPTY_CLOUD, path + ": no vertices");
  return pts;
}

}  // namespace

// geo::load_point_cloud (point_cloud_io.cpp:108-141)
std::vector<V3> load_point_cloud(const std::string& path) {
  std::ifstream in(path);
  if (!in) raise(TG_ERR_IO, "cannot open " + path);
  std::string line;
  size_t line_no = 0;
  std::streampos first_pos = in.tellg();
  while (std::getline(in, line)) {
    ++line_no;
    if (!split_ws(line).empty()) break;
    first_pos = in.tellg();
  }
  const auto toks = split_ws(line);
  if (toks.empty()) raise(TG_ERR_EMPTY_CLOUD, path + ": empty file");
  if (toks[0] == "ply") return load_ply(in, path);
  in.clear();
  in.seekg(first_pos);
  line_no -= 1;
  std::vector<V3> pts;
  while (std::getline(in, line)) {
    ++line_no;
    const auto t = split_ws(line);
    if (t.empty()) continue;
    if (t.size() < 3) cloud_fail(path, line_no, "expected 3 coordinates");
    double x, y, z;
    if (!parse_double(t[0], x) || !parse_double(t[1], y) || !parse_double(t[2], z))
      cloud_fail(path, line_no, "bad coordinate");
    pts.push_back({x * kFileUnitToMeter, y * kFileUnitToMeter, z * kFileUnitToMeter});
  }
  if (pts.empty()) raise(TG_ERR_EMPTY_CLOUD, path + ": no points");
  return pts;
}

// indenter_cloud_for (scene_builder.cpp:33-50): cloud_path, else the
// generated shape, else the object name as a file; subsampled to
// target_points.
std::vector<V3> indenter_cloud_for(const Config& c, const std::string& object) {
  std::vector<V3> cloud;
  if (!c.cloud_path.empty() && (object.empty() || object == c.cloud_path)) {
    cloud = load_point_cloud(c.cloud_path);
  } else {
    const std::string shape = object.empty() ? c.generated_shape : object;
    Shape probe;
    if (!make_shape(shape, probe))
      cloud = load_point_cloud(shape);  // the object name as a file path
    else
      cloud = generate_cloud(shape, c.source_points, c.seed);
  }
  if (c.target_points < cloud.size()) cloud = subsample(cloud, c.target_points, c.seed);
  return cloud;
}

// place_for_press (scene_builder.cpp:48-61).
std::vector<V3> place_for_press(const Config& c, const std::vector<V3>& cloud, double off_x,
                                double off_y) {
  const std::vector<V3> rotated = place(cloud, V3{0, 0, 0}, c.z_rotation_rad);
  V3 lo, hi;
  bbox(rotated, lo, hi);
  const double e = c.edge_mm * 1e-3;
  const double centre = 0.5 * e;
  const double top = 0.5 * e + 0.5 * (c.size_mm[2] * 1e-3);  // elastomer_top_z
  const V3 target{centre + off_x - 0.5 * (lo.x + hi.x), centre + off_y - 0.5 * (lo.y + hi.y),
                  top + c.gap_mm * 1e-3 - lo.z};
  return place(rotated, target, 0.0);
}

std::vector<V3> placed_indenter(const Config& c, const std::string& object, double off_x,
                                double off_y) {
  return place_for_press(c, indenter_cloud_for(c, object), off_x, off_y);
}

// ---- episode setup on the device (f3; setup_kernels.cu) --------------------
}  // namespace tacchi_b200::host
namespace tacchi_b200 {
int device_indenter_cloud(int device, const std::string& shape, uint64_t source_points,
                          uint64_t target_points, uint64_t seed, double** d_cloud, int64_t* n_out);
int device_place_for_press(const double* d_cloud, int64_t n, double z_rotation, double centre,
                           double top_plus_gap, double off_x, double off_y,
                           std::vector<host::V3>& out);
void device_free(void* p);
}  // namespace tacchi_b200
namespace tacchi_b200::host {

// The generated shape indenter_cloud_for would sample for (cfg, object), or
// "" when the indenter comes from a point-cloud file (scene_builder.cpp:33-46).
std::string generated_shape_of(const Config& c, const std::string& object) {
  if (!c.cloud_path.empty() && (object.empty() || object == c.cloud_path)) return "";
  const std::string shape = object.empty() ? c.generated_shape : object;
  Shape probe;
  return make_shape(shape, probe) ? shape : "";
}

// Device builds sample generated indenters on the GPU (TACCHI_HOST_SETUP=1
// keeps the host restatement; both are bit-identical to the reference).
bool device_setup_enabled() {
  const char* e = std::getenv("TACCHI_HOST_SETUP");
  return !(e && std::atoi(e) != 0);
}

// A generated indenter cloud in device memory (indenter_cloud_for), shared
// by the placements of one object.
struct DeviceCloud {
  double* d = nullptr;
  int64_t n = 0;
  DeviceCloud() = default;
  DeviceCloud(const DeviceCloud&) = delete;
  DeviceCloud& operator=(const DeviceCloud&) = delete;
  ~DeviceCloud() {
    if (d) device_free(d);
  }
};

void device_cloud_for(int device, const Config& c, const std::string& shape, DeviceCloud& dc) {
  const int rc = device_indenter_cloud(device, shape, c.source_points, c.target_points, c.seed,
                                       &dc.d, &dc.n);
  if (rc) raise(rc, tg_last_error());
}

std::vector<V3> device_place(const DeviceCloud& dc, const Config& c, double off_x, double off_y) {
  const double e = c.edge_mm * 1e-3;
  const double centre = 0.5 * e;
  const double top = 0.5 * e + 0.5 * (c.size_mm[2] * 1e-3);  // elastomer_top_z
  std::vector<V3> out;
  const int rc = device_place_for_press(dc.d, dc.n, c.z_rotation_rad, centre,
                                        top + c.gap_mm * 1e-3, off_x, off_y, out);
  if (rc) raise(rc, tg_last_error());
  return out;
}

std::shared_ptr<DeviceCloud> device_cloud_for_object(int device, const Config& c,
                                                     const std::string& object) {
  const std::string shape = generated_shape_of(c, object);
  if (shape.empty() || !device_setup_enabled()) return nullptr;
  auto dc = std::make_shared<DeviceCloud>();
  device_cloud_for(device, c, shape, *dc);
  return dc;
}

std::vector<V3> place_for_press_on(const DeviceCloud& dc, const Config& c, double off_x,
                                   double off_y) {
  return device_place(dc, c, off_x, off_y);
}

size_t device_cloud_size(const DeviceCloud& dc) { return static_cast<size_t>(dc.n); }

// placed_indenter for a simulation on `device`: generated shapes are sampled
// and placed on the GPU, point-cloud files on the host.
std::vector<V3> placed_indenter_on(int device, const Config& c, const std::string& object,
                                   double off_x, double off_y) {
  const std::string shape = generated_shape_of(c, object);
  if (shape.empty() || !device_setup_enabled()) return placed_indenter(c, object, off_x, off_y);
  DeviceCloud dc;
  device_cloud_for(device, c, shape, dc);
  return device_place(dc, c, off_x, off_y);
}

// init_scene's checks and particle assembly (scene.cpp:15-87) for
// build_sim's parameters (scene_builder.cpp:63-78).
struct Scene {
  tg_params P{};
  std::vector<double> x, v, mass, vol0;
  std::vector<uint8_t> tag;
  std::vector<uint32_t> surf;
  tg_surface S{};
  int64_t n_el = 0;
  double v0[3] = {0.0, 0.0, 0.0};  // init_scene's indenter_velocity
};

void check_margin(const tg_params& P, const V3& lo, const V3& hi, const char* label) {
  const double margin = 2.0 * P.dx;
  for (int a = 0; a < 3; ++a) {
    const double glo = P.origin[a];
    const double ghi = P.origin[a] + (static_cast<double>(P.res[a]) - 1.0) * P.dx;
    if (lo[a] - glo < margin || ghi - hi[a] < margin)
      raise(TG_ERR_GRID_TOO_SMALL, std::string(label) +
                                       " bounding box violates the 2-node grid margin on axis " +
                                       std::to_string(a));
  }
}

// mpm::init_scene (scene.cpp:28-87) from its own inputs: SceneParams, the
// elastomer lattice (positions in lattice order, or make_elastomer_lattice's
// when `lattice.positions` is NULL) and the placed indenter points.
Scene init_scene_arrays(const tg_scene_params& sp, const tg_lattice& lat,
                        const std::vector<V3>& indenter, const double v0[3]) {
  Scene sc;
  for (int a = 0; a < 3; ++a)
    if (lat.counts[a] < 2) raise(TG_ERR_CONFIG, "make_elastomer_lattice: counts must be >= 2 per axis");
  const int64_t nx = lat.counts[0], ny = lat.counts[1], nz = lat.counts[2];
  const int64_t n_el = nx * ny * nz;
  if (n_el == 0 || indenter.empty())
    raise(TG_ERR_EMPTY_SCENE, "init_scene: both elastomer and indenter particle sets must be non-empty");
  // MaterialParams::validate (material.cpp:11-16), dt (scene.cpp:33)
  if (!(sp.youngs_modulus > 0.0)) raise(TG_ERR_CONFIG, "youngs_modulus must be > 0");
  if (!(sp.poisson_ratio >= 0.0 && sp.poisson_ratio < 0.5))
    raise(TG_ERR_CONFIG, "poisson_ratio must be in [0, 0.5)");
  if (!(sp.density > 0.0)) raise(TG_ERR_CONFIG, "density must be > 0");
  if (!(sp.dt > 0.0)) raise(TG_ERR_CONFIG, "dt must be > 0");
  tg_params& P = sc.P;
  for (int a = 0; a < 3; ++a) {
    P.res[a] = sp.grid_resolution[a];
    P.origin[a] = sp.grid_origin[a];
    P.gravity[a] = sp.gravity[a];
  }
  if (P.res[0] < 4 || P.res[1] < 4 || P.res[2] < 4)
    raise(TG_ERR_CONFIG, "grid resolution must be >= 4 per axis");
  P.dx = sp.grid_edge / P.res[0];  // scene.cpp:41-42
  if (!(P.dx > 0.0)) raise(TG_ERR_CONFIG, "grid spacing must be > 0");
  P.youngs_modulus = sp.youngs_modulus;
  P.poisson_ratio = sp.poisson_ratio;
  P.density = sp.density;
  P.dt = sp.dt;
  if (sp.fixed_bottom_layers < 0) raise(TG_ERR_CONFIG, "fixed_bottom_layers must be >= 0");

  // LatticeMeta::spacing (particle_set.hpp:23-26); make_elastomer_lattice
  double h[3];
  for (int a = 0; a < 3; ++a) h[a] = lat.dims[a] / (lat.counts[a] - 1);
  std::vector<V3> el(static_cast<size_t>(n_el));
  for (int64_t p = 0; p < n_el; ++p) {
    if (lat.positions) {
      el[p] = {lat.positions[3 * p], lat.positions[3 * p + 1], lat.positions[3 * p + 2]};
    } else {
      const int64_t i = p / (ny * nz), j = (p / nz) % ny, k = p % nz;
      el[p] = {lat.origin[0] + i * h[0], lat.origin[1] + j * h[1], lat.origin[2] + k * h[2]};
    }
  }
  V3 lo, hi;
  bbox(el, lo, hi);
  check_margin(P, lo, hi, "elastomer");
  bbox(indenter, lo, hi);
  check_margin(P, lo, hi, "indenter");

  const double el_vol0 = lat.dims[0] * lat.dims[1] * lat.dims[2] / static_cast<double>(n_el);
  const double el_mass = sp.density * el_vol0;
  const double ind_bbox_vol = std::max((hi.x - lo.x) * (hi.y - lo.y) * (hi.z - lo.z), 1e-30);
  const double ind_vol0 = ind_bbox_vol / static_cast<double>(indenter.size());
  const double ind_mass = sp.density * ind_vol0 * sp.indenter_mass_scale;

  const int64_t n = n_el + static_cast<int64_t>(indenter.size());
  sc.n_el = n_el;
  sc.x.resize(3 * n);
  sc.v.assign(3 * n, 0.0);
  sc.mass.assign(n, ind_mass);
  sc.vol0.assign(n, ind_vol0);
  sc.tag.assign(n, 2);  // Tag::Indenter
  // lattice order (i, j, k), k fastest; the bottom layers k < n_fixed are
  // ElastomerBottom (scene.cpp:54-60)
  for (int64_t p = 0; p < n_el; ++p) {
    sc.x[3 * p] = el[p].x;
    sc.x[3 * p + 1] = el[p].y;
    sc.x[3 * p + 2] = el[p].z;
    sc.mass[p] = el_mass;
    sc.vol0[p] = el_vol0;
    sc.tag[p] = (p % nz) < sp.fixed_bottom_layers ? 1 : 0;
  }
  for (size_t q = 0; q < indenter.size(); ++q) {
    const int64_t p = n_el + static_cast<int64_t>(q);
    sc.x[3 * p] = indenter[q].x;
    sc.x[3 * p + 1] = indenter[q].y;
    sc.x[3 * p + 2] = indenter[q].z;
    for (int a = 0; a < 3; ++a) sc.v[3 * p + a] = v0[a];
  }
  for (int a = 0; a < 3; ++a) sc.v0[a] = v0[a];
  // SurfaceLattice (scene.cpp:71-84): the top layer k = nz - 1
  sc.surf.resize(nx * ny);
  for (int64_t i = 0; i < nx; ++i)
    for (int64_t j = 0; j < ny; ++j)
      sc.surf[i * ny + j] = static_cast<uint32_t>((i * ny + j) * nz + (nz - 1));
  sc.S.nx = static_cast<int>(nx);
  sc.S.ny = static_cast<int>(ny);
  sc.S.x0 = lat.origin[0];
  sc.S.y0 = lat.origin[1];
  sc.S.sx = h[0];
  sc.S.sy = h[1];
  sc.S.z0 = lat.origin[2] + lat.dims[2];
  sc.S.particle = sc.surf.data();
  return sc;
}

// build_sim's SceneParams and elastomer_for(cfg) (scene_builder.cpp:13-31,
// 63-78) around init_scene.
Scene build_scene(const Config& c, const std::vector<V3>& indenter) {
  tg_scene_params sp{};
  const double edge = c.edge_mm * 1e-3;
  tg_lattice lat{};
  for (int a = 0; a < 3; ++a) {
    sp.grid_resolution[a] = c.nodes[a];
    sp.grid_origin[a] = 0.0;
    lat.counts[a] = c.counts[a];
    lat.dims[a] = c.size_mm[a] * 1e-3;
    lat.origin[a] = 0.5 * edge - 0.5 * lat.dims[a];
  }
  sp.grid_edge = edge;
  sp.youngs_modulus = c.E;
  sp.poisson_ratio = c.nu;
  sp.density = c.rho;
  sp.dt = c.dt;
  sp.fixed_bottom_layers = c.fixed_bottom_layers;
  sp.gravity[0] = 0.0;
  sp.gravity[1] = 0.0;
  sp.gravity[2] = -c.gravity_mps2;
  sp.indenter_mass_scale = c.rigid_mass_scale;
  const double zero[3] = {0.0, 0.0, 0.0};  // build_sim passes no velocity
  return init_scene_arrays(sp, lat, indenter, zero);
}

int create_from(int device, Scene& sc, tg_handle* out) {
  tg_particles tp{};
  tp.n = static_cast<int64_t>(sc.mass.size());
  tp.n_elastomer = sc.n_el;
  tp.x = sc.x.data();
  tp.v = sc.v.data();
  tp.mass = sc.mass.data();
  tp.volume0 = sc.vol0.data();
  tp.tag = sc.tag.data();
  for (int a = 0; a < 3; ++a) tp.indenter_velocity[a] = sc.v0[a];
  return tg_create(device, &sc.P, &tp, &sc.S, out);
}

int build_sim_from(int device, const Config& c, const std::vector<V3>& placed, tg_handle* out) {
  Scene sc = build_scene(c, placed);
  int rc = create_from(device, sc, out);
  // SceneConfig::deterministic (scene_config.hpp:78, default true): the
  // reference is bit-reproducible by construction; here it selects the
  // fixed-point node accumulation (SPEC "Concurrency Model")
  if (!rc && c.deterministic) {
    rc = tg_set_deterministic(*out, 1);
    if (rc) {
      tg_destroy(*out);
      *out = nullptr;
    }
  }
  return rc;
}

namespace {
json v3j(const double* v) { return json::array({v[0], v[1], v[2]}); }
json v3ij(const int* v) { return json::array({v[0], v[1], v[2]}); }
}  // namespace

// to_json_string (scene_config.cpp:124-170): 2-space indented + newline.
std::string to_json_string(const Config& c) {
  json j;
  j["elastomer"] = {{"size_mm", v3j(c.size_mm)},
                    {"particle_counts", v3ij(c.counts)},
                    {"youngs_modulus_pa", c.E},
                    {"poisson_ratio", c.nu},
                    {"density_kg_m3", c.rho},
                    {"fixed_bottom_layers", c.fixed_bottom_layers}};
  j["grid"] = {{"nodes_per_axis", v3ij(c.nodes)}, {"edge_mm", c.edge_mm}};
  j["time"] = {{"dt_s", c.dt},
               {"substeps_per_control_step", c.substeps_per_control_step},
               {"press_speed_mm_s", c.press_speed_mm_s}};
  j["indenter"] = {{"cloud_path", c.cloud_path},
                   {"generated_shape", c.generated_shape},
                   {"source_points", c.source_points},
                   {"target_points", c.target_points},
                   {"seed", c.seed},
                   {"gap_mm", c.gap_mm},
                   {"z_rotation_rad", c.z_rotation_rad},
                   {"rigid_mass_scale", c.rigid_mass_scale}};
  j["press_grid"] = {{"positions_x", c.positions_x},
                     {"positions_y", c.positions_y},
                     {"step_mm", c.step_mm},
                     {"depths_mm", c.depths_mm}};
  j["lights"] = json::array();
  for (const Light& l : c.lights)
    j["lights"].push_back({{"direction", v3j(l.dir)},
                           {"diffuse_rgb", v3j(l.diffuse)},
                           {"specular_rgb", v3j(l.specular)}});
  j["render"] = {{"ambient_k", c.ka},
                 {"diffuse_k", c.kd},
                 {"specular_k", c.ks},
                 {"shininess", c.shininess},
                 {"ambient_rgb", v3j(c.ambient)},
                 {"view_dir", v3j(c.view)},
                 {"pixel_to_meter", c.pixel_to_meter},
                 {"image_width", c.image_w},
                 {"image_height", c.image_h},
                 {"background_image", c.background_image}};
  j["alignment"] = json::object();
  for (const auto& [name, a] : c.alignment)
    j["alignment"][name] = {{"offset_px", json::array({a.ox, a.oy})}, {"scale", a.scale}};
  j["objects"] = c.objects;
  j["output_dir"] = c.output_dir;
  j["deterministic"] = c.deterministic;
  j["workers"] = c.workers;
  j["gravity_mps2"] = c.gravity_mps2;
  return j.dump(2) + "\n";
}

// Background images of render configs, decoded once per (path, size, mtime)
// and kept for the process (tg_render::background points into the cache).
const uint8_t* background_pixels(const std::string& path, int& w, int& h) {
  struct Entry {
    std::vector<uint8_t> rgb;
    int w = 0, h = 0;
    std::uintmax_t size = 0;
    std::filesystem::file_time_type mtime{};
  };
  static std::mutex mu;
  static std::map<std::string, std::unique_ptr<Entry>> cache;
  static std::vector<std::unique_ptr<Entry>> retired;  // earlier tg_render may still point here
  std::error_code ec;
  const auto size = std::filesystem::file_size(path, ec);
  if (ec) raise(TG_ERR_IO, "cannot open " + path);
  const auto mtime = std::filesystem::last_write_time(path, ec);
  std::lock_guard<std::mutex> lk(mu);
  auto& e = cache[path];
  if (!e || e->size != size || e->mtime != mtime) {
    auto fresh = std::make_unique<Entry>();
    fresh->rgb = load_png(path, fresh->w, fresh->h);
    fresh->size = size;
    fresh->mtime = mtime;
    if (e) retired.push_back(std::move(e));
    e = std::move(fresh);
  }
  w = e->w;
  h = e->h;
  return e->rgb.data();
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const HostError& e) {
    return fail(e.code, e.msg);
  } catch (const std::exception& e) {
    return fail(TG_ERR_CONFIG, e.what());
  }
}

}  // namespace tacchi_b200::host

using namespace tacchi_b200::host;

extern "C" {

int tg_build_sim(int device, const char* config_json, const char* object, double offset_x,
                 double offset_y, tg_handle* out) {
  return guarded([&] {
    const Config c = parse_config(config_json);
    return build_sim_from(device, c,
                          placed_indenter_on(device, c, object ? object : "", offset_x, offset_y),
                          out);
  });
}

int tg_init_scene(int device, const tg_scene_params* params, const tg_lattice* elastomer,
                  const double* indenter, int64_t n_indenter, const double indenter_velocity[3],
                  tg_handle* out) {
  return guarded([&] {
    if (!params || !elastomer || !out || (n_indenter > 0 && !indenter))
      raise(TG_ERR_INVALID_ARGUMENT, "tg_init_scene: null argument");
    std::vector<V3> ind(static_cast<size_t>(std::max<int64_t>(n_indenter, 0)));
    for (size_t q = 0; q < ind.size(); ++q) ind[q] = {indenter[3 * q], indenter[3 * q + 1], indenter[3 * q + 2]};
    const double zero[3] = {0.0, 0.0, 0.0};
    Scene sc = init_scene_arrays(*params, *elastomer, ind, indenter_velocity ? indenter_velocity : zero);
    return create_from(device, sc, out);
  });
}

int tg_build_sim_points(int device, const char* config_json, const double* indenter,
                        int64_t n_indenter, tg_handle* out) {
  return guarded([&] {
    if (!out || (n_indenter > 0 && !indenter))
      raise(TG_ERR_INVALID_ARGUMENT, "tg_build_sim_points: null argument");
    const Config c = parse_config(config_json);
    std::vector<V3> placed(static_cast<size_t>(std::max<int64_t>(n_indenter, 0)));
    for (size_t q = 0; q < placed.size(); ++q)
      placed[q] = {indenter[3 * q], indenter[3 * q + 1], indenter[3 * q + 2]};
    return build_sim_from(device, c, placed, out);
  });
}

// Many episodes of one object (config 4, the harness's positions): the
// indenter cloud (rejection sampling + subsample, the expensive part) is
// generated once and shared; each episode gets its own z-rotation and
// lateral offset (place_for_press, scene_builder.cpp:48-61) and simulation.
// Built on host threads; on failure every handle created so far is destroyed.
int tg_build_episodes(int device, const char* config_json, const char* object, int n_episodes,
                      const double* poses, tg_handle* out) {
  return guarded([&] {
    if (n_episodes < 0 || (n_episodes > 0 && (!poses || !out)))
      raise(TG_ERR_INVALID_ARGUMENT, "tg_build_episodes: bad argument");
    const Config base = parse_config(config_json);
    const std::string obj = object ? object : "";
    // the cloud once per object: on the device for a generated shape
    const std::string shape = generated_shape_of(base, obj);
    const bool on_device = !shape.empty() && device_setup_enabled();
    DeviceCloud dcloud;
    std::vector<V3> cloud;
    if (on_device) device_cloud_for(device, base, shape, dcloud);
    else cloud = indenter_cloud_for(base, obj);
    std::vector<int> rc(static_cast<size_t>(n_episodes), TG_OK);
    std::vector<std::string> msg(static_cast<size_t>(n_episodes));
    std::atomic<int> next{0};
    auto worker = [&] {
      for (int e; (e = next.fetch_add(1)) < n_episodes;) {
        out[e] = nullptr;
        try {
          Config c = base;
          c.z_rotation_rad = poses[3 * e + 2];
          const std::vector<V3> placed =
              on_device ? device_place(dcloud, c, poses[3 * e], poses[3 * e + 1])
                        : place_for_press(c, cloud, poses[3 * e], poses[3 * e + 1]);
          rc[e] = build_sim_from(device, c, placed, &out[e]);
          if (rc[e]) msg[e] = tg_last_error();
        } catch (const HostError& err) {
          rc[e] = err.code;
          msg[e] = err.msg;
        }
      }
    };
    const unsigned hw = std::thread::hardware_concurrency();
    const int nt = std::max(1, std::min<int>(n_episodes, static_cast<int>(std::min(8u, hw ? hw : 4u))));
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    for (int e = 0; e < n_episodes; ++e)
      if (rc[e]) {
        for (int k = 0; k < n_episodes; ++k)
          if (out[k]) {
            tg_destroy(out[k]);
            out[k] = nullptr;
          }
        raise(rc[e], msg[e]);
      }
    return TG_OK;
  });
}

int tg_render_from_config(const char* config_json, const char* object, tg_render* r) {
  return guarded([&] {
    const Config c = parse_config(config_json);
    const uint8_t* background = nullptr;
    if (!c.background_image.empty()) {
      // render_params_struct loads the PNG (scene_config.cpp:77-78); phong
      // requires its size to be the image's (phong.cpp:46-48)
      int bw = 0, bh = 0;
      background = background_pixels(c.background_image, bw, bh);
      if (bw != c.image_w || bh != c.image_h)
        raise(TG_ERR_SHAPE_MISMATCH, "phong_render: background image size differs from the depth map");
    }
    std::memset(r, 0, sizeof(*r));
    r->pixel_to_meter = c.pixel_to_meter;
    const auto it = c.alignment.find(object ? object : "");
    const Config::Align a = it == c.alignment.end() ? Config::Align{} : it->second;
    r->crop_offset[0] = a.ox;
    r->crop_offset[1] = a.oy;
    r->crop_scale = a.scale;
    r->width = c.image_w;
    r->height = c.image_h;
    r->ambient_k = c.ka;
    r->diffuse_k = c.kd;
    r->specular_k = c.ks;
    r->shininess = c.shininess;
    for (int k = 0; k < 3; ++k) {
      r->ambient_rgb[k] = c.ambient[k];
      r->view_dir[k] = c.view[k];
    }
    if (c.lights.empty() || c.lights.size() > 8)
      raise(TG_ERR_CONFIG, "phong_render: between 1 and 8 light sources required");
    r->n_lights = static_cast<int>(c.lights.size());
    for (size_t l = 0; l < c.lights.size(); ++l)
      for (int k = 0; k < 3; ++k) {
        r->lights[l][k] = c.lights[l].dir[k];
        r->lights[l][3 + k] = c.lights[l].diffuse[k];
        r->lights[l][6 + k] = c.lights[l].specular[k];
      }
    r->background = background;
    return TG_OK;
  });
}

int tg_generate_cloud(const char* shape, int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    const std::vector<V3> pts = generate_cloud(shape ? shape : "", static_cast<size_t>(n), seed);
    for (size_t i = 0; i < pts.size(); ++i) {
      out[3 * i] = pts[i].x;
      out[3 * i + 1] = pts[i].y;
      out[3 * i + 2] = pts[i].z;
    }
    return TG_OK;
  });
}

int tg_placed_indenter(const char* config_json, const char* object, double offset_x,
                       double offset_y, double* out, int64_t* n) {
  return guarded([&] {
    const Config c = parse_config(config_json);
    const std::vector<V3> pts = placed_indenter(c, object ? object : "", offset_x, offset_y);
    *n = static_cast<int64_t>(pts.size());
    if (out)
      for (size_t i = 0; i < pts.size(); ++i) {
        out[3 * i] = pts[i].x;
        out[3 * i + 1] = pts[i].y;
        out[3 * i + 2] = pts[i].z;
      }
    return TG_OK;
  });
}

}  // extern "C"
