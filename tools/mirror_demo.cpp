// mirror_demo — exercises the C++ mirror (include/tacchi_b200.hpp) the way a
// reference caller that owns its geometry would: mpm::init_scene from
// SceneParams + an elastomer lattice + its own indenter points
// (sim_state.hpp:102-104), sim::build_sim(cfg, points) (scene_builder.hpp:29-30),
// the post-step grid (set_keep_grid + grid_window + grid) and the per-particle
// constants. Prints one JSON line; tests/test_gpu_parity.py checks it.
//
//   mirror_demo
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "tacchi_b200.hpp"

using tacchi_b200::Vec3;

int main() {
  try {
    // the SMALL test scene (tests/scenes.py): 31 x 31 x 7 gel, 6 x 6 x 1.2 mm,
    // on a 64^3 grid of 12 mm, with a 3000-point sphere2 indenter 20 um above
    const std::string cfg =
        "{\"elastomer\": {\"size_mm\": [6, 6, 1.2], \"particle_counts\": [31, 31, 7]},"
        " \"grid\": {\"nodes_per_axis\": [64, 64, 64], \"edge_mm\": 12.0},"
        " \"time\": {\"dt_s\": 2e-6},"
        " \"render\": {\"image_width\": 160, \"image_height\": 120},"
        " \"indenter\": {\"generated_shape\": \"sphere2\", \"source_points\": 20000,"
        " \"target_points\": 3000, \"gap_mm\": 0.02}}";
    int64_t n = 0;
    tacchi_b200::check(tg_placed_indenter(cfg.c_str(), "", 0.0, 0.0, nullptr, &n));
    std::vector<Vec3> pts(static_cast<size_t>(n));
    tacchi_b200::check(tg_placed_indenter(cfg.c_str(), "", 0.0, 0.0, pts.front().data(), &n));

    // (1) build_sim with the caller's points == the config path
    auto a = tacchi_b200::sim::build_sim(cfg, pts);
    auto b = tacchi_b200::sim::build_sim(cfg, "");
    std::vector<double> xa, xb;
    a.download(&xa, nullptr, nullptr, nullptr);
    b.download(&xb, nullptr, nullptr, nullptr);
    const bool same_setup = xa == xb;

    // (2) init_scene from its own inputs, the same scene as the config path
    // (the config's millimetres converted as SceneConfig does: mm * 1e-3)
    const double edge = 12.0 * 1e-3;
    tacchi_b200::mpm::SceneParams p;
    p.grid_resolution = {64, 64, 64};
    p.grid_edge = edge;
    p.dt = 2e-6;
    tacchi_b200::mpm::ElastomerLattice gel;
    gel.counts = {31, 31, 7};
    gel.dims = {6.0 * 1e-3, 6.0 * 1e-3, 1.2 * 1e-3};
    for (int a = 0; a < 3; ++a) gel.origin[a] = 0.5 * edge - 0.5 * gel.dims[a];  // elastomer_for
    auto s = tacchi_b200::mpm::init_scene(p, gel, pts);
    std::vector<double> xs;
    s.download(&xs, nullptr, nullptr, nullptr);
    const bool same_init = xs == xb;
    std::vector<double> mass, vol;
    std::vector<uint8_t> tag;
    s.constants(&mass, &vol, &tag);
    double total_mass = 0.0;
    for (double m : mass) total_mass += m;

    // (3) step with the post-step grid kept; the grid holds the last
    // substep's P2G (mass conserved over the active window)
    s.set_keep_grid(true);
    tacchi_b200::mpm::step(s, Vec3{0.0, 0.0, -0.05}, 20);
    const auto w = s.grid_window();
    const auto g = s.grid(w[0], w[1]);
    double grid_mass = 0.0;
    for (double m : g.mass) grid_mass += m;

    // (4) capture with render inputs resolved once
    const auto rs = tacchi_b200::sim::RenderSetup::from_config(cfg, "");
    const auto cap = tacchi_b200::sim::capture(s, rs);
    double max_depth = 0.0;
    for (double d : cap.depth.values) max_depth = d > max_depth ? d : max_depth;

    std::printf("{\"same_setup\": %s, \"same_init\": %s, \"particles\": %lld, \"step_count\": %lld, "
                "\"total_mass\": %.17g, \"grid_mass\": %.17g, \"window\": [%d, %d, %d, %d, %d, %d], "
                "\"image\": [%d, %d], \"max_depth_m\": %.17g}\n",
                same_setup ? "true" : "false", same_init ? "true" : "false",
                static_cast<long long>(s.size()), static_cast<long long>(s.step_count()),
                total_mass, grid_mass, w[0][0], w[0][1], w[0][2], w[1][0], w[1][1], w[1][2],
                cap.image.width, cap.image.height, max_depth);
  } catch (const tacchi_b200::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}
