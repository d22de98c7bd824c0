// Host-side SceneConfig restatement shared by the setup path (host_setup.cpp)
// and the bridge Session (bridge.cpp). Field names and defaults follow
// /root/reference/proj/include/tacchi/config/scene_config.hpp:19-94.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "tacchi_cuda.h"

namespace tacchi_b200::host {

struct HostError {
  int code;
  std::string msg;
};

[[noreturn]] void raise(int code, const std::string& msg);

struct V3 {
  double x = 0, y = 0, z = 0;
  double operator[](int a) const { return a == 0 ? x : (a == 1 ? y : z); }
};

struct Light {
  double dir[3], diffuse[3], specular[3];
};

struct Config {
  double size_mm[3] = {20.0, 20.0, 4.0};
  int counts[3] = {101, 101, 21};
  double E = 1.45e5, nu = 0.45, rho = 1000.0;
  int fixed_bottom_layers = 2;
  int nodes[3] = {256, 256, 256};
  double edge_mm = 33.0;
  double dt = 1e-4;
  int substeps_per_control_step = 10;
  double press_speed_mm_s = 10.0;
  std::string cloud_path, generated_shape = "sphere";
  uint64_t source_points = 1000000, target_points = 100000, seed = 20230115;
  double gap_mm = 0.1, z_rotation_rad = 0.0, rigid_mass_scale = 80.0;
  int positions_x = 3, positions_y = 3;
  double step_mm = 1.0;
  std::vector<double> depths_mm = {0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0};
  std::vector<Light> lights;
  double ka = 1.0, kd = 0.55, ks = 0.25, shininess = 24.0;
  double ambient[3] = {0.34, 0.37, 0.44};
  double view[3] = {0, 0, -1};
  double pixel_to_meter = 2.8125e-5;
  int image_w = 640, image_h = 480;
  std::string background_image;
  struct Align {
    double ox = 0, oy = 0, scale = 1.0;
  };
  std::map<std::string, Align> alignment;
  std::vector<std::string> objects = {"sphere"};
  std::string output_dir = "tacchi_out";
  bool deterministic = true;
  int workers = 0;
  double gravity_mps2 = 0.0;
};

// from_json_string (scene_config.cpp:187-257): partial overrides of
// default_config(). Throws HostError{TG_ERR_CONFIG, ...}.
// geo::is_known_shape (shapes.cpp:226-229).
bool is_known_shape(const std::string& name);

Config parse_config(const char* text);

// render::save_png (image.cpp:23-49; 8-bit RGB, zlib, filter "none") and
// render::save_depth_map (depth_map.cpp:28-38; JSON header line + float32).
void save_png(const std::string& path, int w, int h, const uint8_t* rgb);
void save_depth_map(const std::string& path, int w, int h, double pixel_to_meter,
                    const double* values);
// render::load_png (image.cpp:51-90): any non-interlaced 8/16-bit PNG ->
// 8-bit RGB (palette / grey expanded, alpha stripped).
std::vector<uint8_t> load_png(const std::string& path, int& w, int& h);

// SceneConfig::validate (scene_config.cpp:83-116, material.cpp:11-16).
void validate(const Config& c);

// to_json_string (scene_config.cpp:124-170), byte-identical output.
std::string to_json_string(const Config& c);

// sim::indenter_cloud_for / place_for_press (scene_builder.cpp:33-61).
std::vector<V3> indenter_cloud_for(const Config& c, const std::string& object);
std::vector<V3> place_for_press(const Config& c, const std::vector<V3>& cloud, double off_x,
                                double off_y);

// Episode setup on the device (setup_kernels.cu, §8 row f3): a generated
// indenter cloud (indenter_cloud_for) in device memory, shared by the
// placements of one object; null when the object is a point-cloud file or
// TACCHI_HOST_SETUP=1 selects the host restatement.
struct DeviceCloud;
std::shared_ptr<DeviceCloud> device_cloud_for_object(int device, const Config& c,
                                                     const std::string& object);
// place_for_press (scene_builder.cpp:48-61) of a device cloud -> host points.
std::vector<V3> place_for_press_on(const DeviceCloud& dc, const Config& c, double off_x,
                                   double off_y);
size_t device_cloud_size(const DeviceCloud& dc);

// sim::build_sim (scene_builder.cpp:63-78) from an already placed indenter.
int build_sim_from(int device, const Config& c, const std::vector<V3>& placed, tg_handle* out);

}  // namespace tacchi_b200::host
