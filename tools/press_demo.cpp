// press_demo — a C++ caller of the B200 path through tacchi_b200.hpp, shaped
// like the reference's bridge::Session control loop (session.cpp:61-98):
// one control step = mpm::step(state, v, substeps_per_control_step) followed
// by sim::capture. Prints one JSON line per run.
//
//   press_demo [config_json] [control_steps]
#include <chrono>
#include <cstdio>
#include <string>

#include "tacchi_b200.hpp"

int main(int argc, char** argv) {
  const std::string cfg = argc > 1 ? argv[1] : "{\"time\": {\"dt_s\": 2e-6}}";
  const int steps = argc > 2 ? std::atoi(argv[2]) : 10;
  try {
    auto state = tacchi_b200::sim::build_sim(cfg, "");
    const auto render = tacchi_b200::sim::RenderSetup::from_config(cfg, "");
    const tacchi_b200::Vec3 v = {0.0, 0.0, -0.01};
    double max_depth = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < steps; ++k) {
      tacchi_b200::mpm::step(state, v, 10);
      const auto cap = tacchi_b200::sim::capture(state, render);
      for (double d : cap.depth.values) max_depth = d > max_depth ? d : max_depth;
    }
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    const auto d = state.diag();
    std::printf("{\"particles\": %lld, \"control_steps\": %d, \"ms_per_control_step\": %.4f, "
                "\"step_count\": %lld, \"min_det_f\": %.17g, \"max_speed\": %.17g, "
                "\"max_depth_m\": %.17g}\n",
                static_cast<long long>(state.size()), steps, ms / steps,
                static_cast<long long>(state.step_count()), d.min_det_f, d.max_speed, max_depth);
  } catch (const tacchi_b200::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}
