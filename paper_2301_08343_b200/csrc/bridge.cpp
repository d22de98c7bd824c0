// Bridge (§8(f) row f1): the reference's co-simulation Session and its
// newline-delimited JSON protocol "tacchi/1" (session.cpp:15-98,
// server.cpp:49-182), driving the B200 hot path. Host C++ over the C-ABI.
//
// A Session owns one device simulation; each control step runs
// mpm::step(state, v, substeps_per_control_step) on the GPU and, on request,
// the fused capture kernel, then writes the PNG and .depth files and a line
// of steps.jsonl exactly as the reference does.
#include <sys/socket.h>
#include <unistd.h>
#include <arpa/inet.h>
#include <netinet/in.h>
#include <zlib.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <limits>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "host_config.hpp"
#include "tacchi_cuda.h"

namespace tacchi_b200 {
int fail(int code, const std::string& msg);
}

namespace tacchi_b200::bridge {

using host::HostError;
using json = nlohmann::json;

namespace {

constexpr const char* kProtocolVersion = "tacchi/1";

void check(int rc) {
  if (rc != TG_OK) throw HostError{rc, tg_last_error()};
}

}  // namespace

}  // namespace tacchi_b200::bridge

namespace tacchi_b200::host {

// ---- SceneConfig::validate (scene_config.cpp:83-116, material.cpp:11-16) -----

void validate(const host::Config& c) {
  auto bad = [](const std::string& m) { throw HostError{TG_ERR_CONFIG, m}; };
  if (!(c.E > 0.0)) bad("youngs_modulus must be > 0");
  if (!(c.nu >= 0.0 && c.nu < 0.5)) bad("poisson_ratio must be in [0, 0.5)");
  if (!(c.rho > 0.0)) bad("density must be > 0");
  for (int a = 0; a < 3; ++a) {
    if (c.counts[a] < 2) bad("elastomer.particle_counts must be >= 2 per axis");
    if (!(c.size_mm[a] > 0.0)) bad("elastomer.size_mm must be positive");
    if (c.nodes[a] < 8) bad("grid.nodes_per_axis must be >= 8");
  }
  if (!(c.edge_mm > 0.0)) bad("grid.edge_mm must be positive");
  if (!(c.dt > 0.0)) bad("time.dt_s must be positive");
  if (c.substeps_per_control_step < 1) bad("time.substeps_per_control_step must be >= 1");
  if (!(c.press_speed_mm_s > 0.0)) bad("time.press_speed_mm_s must be positive");
  if (c.target_points < 1) bad("indenter.target_points must be >= 1");
  if (c.cloud_path.empty() && !is_known_shape(c.generated_shape))
    bad("indenter: no cloud_path and unknown generated_shape '" + c.generated_shape + "'");
  if (c.positions_x < 1 || c.positions_y < 1) bad("press grid must have at least one position");
  if (c.depths_mm.empty()) bad("press.depths_mm must not be empty");
  if (c.lights.empty()) bad("at least one light source required");
  if (c.image_w < 2 || c.image_h < 2) bad("render image size too small");
  if (!(c.pixel_to_meter > 0.0)) bad("pixel_to_meter must be positive");
  if (c.fixed_bottom_layers < 0 || c.fixed_bottom_layers >= c.counts[2])
    bad("elastomer.fixed_bottom_layers out of range");
  const double dx = c.edge_mm * 1e-3 / c.nodes[0];
  const double bound = 0.5 * dx / std::sqrt(c.E / c.rho);  // scene.cpp:9-11
  if (c.dt > bound)
    std::cerr << "[tacchi] warning: dt_s = " << c.dt
              << " exceeds the stability bound 0.5*dx/sqrt(E/rho) = " << bound
              << "; explicit stepping may diverge at this grid resolution\n";
}

}  // namespace tacchi_b200::host

namespace tacchi_b200::bridge {

using host::save_depth_map;
using host::save_png;
using host::validate;

// ---- Session (session.hpp:61-77) -----------------------------------------------

enum class CommandMode { Velocity, Position };

struct StepCommand {
  CommandMode mode = CommandMode::Velocity;
  double vector[3] = {0, 0, 0};
  double sim_time = std::numeric_limits<double>::quiet_NaN();
  bool request_image = false;
};

struct StepReply {
  int64_t step_index = 0;
  double depth_m = 0.0;
  bool terminal = false;
  std::string image_path, depth_map_path;
};

struct TerminalCondition {
  double max_depth_m = std::numeric_limits<double>::infinity();
  int64_t max_steps = 0;
  bool any_bound() const {
    return max_depth_m < std::numeric_limits<double>::infinity() || max_steps > 0;
  }
};

class Session {
 public:
  Session(const std::string& config_json, std::filesystem::path dir, std::string object,
          TerminalCondition term, int device)
      : dir_(std::move(dir)), object_(std::move(object)), term_(term) {
    cfg_ = host::parse_config(config_json.c_str());
    validate(cfg_);
    if (!term_.any_bound()) {
      double deepest = 0.0;
      for (double d : cfg_.depths_mm) deepest = std::max(deepest, d);
      term_.max_depth_m = deepest * 1e-3;
    }
    gap_m_ = cfg_.gap_mm * 1e-3;
    check(tg_build_sim(device, config_json.c_str(), object_.c_str(), 0.0, 0.0, &h_));
    check(tg_render_from_config(config_json.c_str(), object_.c_str(), &render_));
    check(tg_capture_buffers(h_, &render_, &cap_depth_, &cap_rgb_));
    std::filesystem::create_directories(dir_);
  }
  ~Session() {
    if (h_) tg_destroy(h_);
  }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  int64_t particles() const { return tg_num_particles(h_); }
  const host::Config& cfg() const { return cfg_; }
  const std::filesystem::path& dir() const { return dir_; }
  int64_t control_steps() const { return control_steps_; }
  double control_dt() const { return cfg_.dt * cfg_.substeps_per_control_step; }
  double depth() const { return std::max(0.0, -offset_[2] - gap_m_); }

  // session.cpp:61-98
  StepReply handle_command(const StepCommand& cmd) {
    if (!h_) throw HostError{TG_ERR_SESSION_NOT_INITIALIZED, "session has no scene"};
    for (double c : cmd.vector)
      if (!std::isfinite(c)) throw HostError{TG_ERR_PROTOCOL, "step vector must be finite"};
    if (!std::isnan(cmd.sim_time)) {
      if (cmd.sim_time < last_sim_time_ - 1e-12)
        throw HostError{TG_ERR_NON_MONOTONIC_TIME, "sim_time " + std::to_string(cmd.sim_time) +
                                                       " decreased (last " +
                                                       std::to_string(last_sim_time_) + ")"};
      last_sim_time_ = cmd.sim_time;
    }
    if (terminal_) {  // physics frozen: repeat the terminal state
      StepReply r = last_reply_;
      r.terminal = true;
      return r;
    }
    const double dtc = control_dt();
    double v[3];
    for (int a = 0; a < 3; ++a)
      v[a] = cmd.mode == CommandMode::Velocity ? cmd.vector[a] : (cmd.vector[a] - offset_[a]) / dtc;
    // mpm::step, and sim::capture when an image is requested, with one sync
    if (cmd.request_image)
      check(tg_step_capture(h_, v, cfg_.substeps_per_control_step, &render_, cap_depth_, cap_rgb_));
    else
      check(tg_step(h_, v, cfg_.substeps_per_control_step));
    for (int a = 0; a < 3; ++a)
      offset_[a] = cmd.mode == CommandMode::Position ? cmd.vector[a] : offset_[a] + v[a] * dtc;
    ++control_steps_;
    if (depth() >= term_.max_depth_m - 1e-12) terminal_ = true;
    if (term_.max_steps > 0 && control_steps_ >= term_.max_steps) terminal_ = true;
    last_reply_ = make_reply(cmd.request_image);
    return last_reply_;
  }

 private:
  // session.cpp:36-58
  StepReply make_reply(bool request_image) {
    StepReply reply;
    reply.step_index = control_steps_;
    reply.depth_m = depth();
    reply.terminal = terminal_;
    if (request_image) {  // captured by handle_command into the pinned buffers
      const int w = render_.width, h = render_.height;
      char name[64];
      std::snprintf(name, sizeof(name), "step_%06lld", static_cast<long long>(control_steps_));
      reply.image_path = (dir_ / (std::string(name) + ".png")).string();
      reply.depth_map_path = (dir_ / (std::string(name) + ".depth")).string();
      save_png(reply.image_path, w, h, cap_rgb_);
      save_depth_map(reply.depth_map_path, w, h, render_.pixel_to_meter * render_.crop_scale,
                     cap_depth_);
    }
    std::ofstream log(dir_ / "steps.jsonl", std::ios::app);
    const json j = {{"step", reply.step_index},
                    {"depth_m", reply.depth_m},
                    {"terminal", reply.terminal},
                    {"image", reply.image_path},
                    {"depth_map", reply.depth_map_path}};
    log << j.dump() << '\n';
    return reply;
  }

  host::Config cfg_;
  std::filesystem::path dir_;
  std::string object_;
  TerminalCondition term_;
  tg_handle h_ = nullptr;
  tg_render render_{};
  double* cap_depth_ = nullptr;  // the handle's pinned capture buffers
  uint8_t* cap_rgb_ = nullptr;
  double offset_[3] = {0, 0, 0};
  double gap_m_ = 0.0;
  double last_sim_time_ = -std::numeric_limits<double>::infinity();
  int64_t control_steps_ = 0;
  bool terminal_ = false;
  StepReply last_reply_;
};

// ---- protocol (server.cpp:49-113) ----------------------------------------------

using LineReader = std::function<bool(std::string&)>;
using LineWriter = std::function<void(const std::string&)>;

namespace {

json error_reply(const std::string& error, const std::string& message, const std::string& echo) {
  return {{"type", "error"}, {"error", error}, {"message", message}, {"echo", echo}};
}

StepCommand parse_step(const json& j) {
  StepCommand cmd;
  const std::string mode = j.value("mode", "velocity");
  if (mode == "velocity")
    cmd.mode = CommandMode::Velocity;
  else if (mode == "position")
    cmd.mode = CommandMode::Position;
  else
    throw HostError{TG_ERR_PROTOCOL, "unknown step mode '" + mode + "'"};
  if (!j.contains("vector") || !j["vector"].is_array() || j["vector"].size() != 3)
    throw HostError{TG_ERR_PROTOCOL, "step requires a 3-element 'vector'"};
  for (int a = 0; a < 3; ++a) cmd.vector[a] = j["vector"][a].get<double>();
  if (j.contains("sim_time")) cmd.sim_time = j["sim_time"].get<double>();
  cmd.request_image = j.value("request_image", false);
  return cmd;
}

std::string read_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw HostError{TG_ERR_IO, "cannot open config " + path};
  return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

}  // namespace

void run_protocol(const LineReader& read_line, const LineWriter& write_line,
                  const std::string& base_config_json, const std::string& session_root,
                  int device) {
  std::unique_ptr<Session> session;
  int session_counter = 0;
  std::string line;
  while (read_line(line)) {
    if (line.empty()) continue;
    json msg = json::parse(line, nullptr, false);
    if (msg.is_discarded()) {
      write_line(error_reply("ProtocolError", "not valid JSON", line).dump());
      continue;
    }
    const std::string type = msg.value("type", "");
    try {
      if (type == "init") {
        std::string cfg = base_config_json;
        if (msg.contains("config_path")) cfg = read_file(msg["config_path"].get<std::string>());
        if (msg.contains("config")) cfg = msg["config"].dump();
        const std::string object = msg.value("object", "");
        TerminalCondition term;
        if (msg.contains("max_depth_m")) term.max_depth_m = msg["max_depth_m"].get<double>();
        if (msg.contains("max_steps")) term.max_steps = msg["max_steps"].get<int64_t>();
        std::string dir = msg.value("session_dir", "");
        if (dir.empty()) dir = session_root + "/session_" + std::to_string(session_counter++);
        session = std::make_unique<Session>(cfg, dir, object, term, device);
        write_line(json{{"type", "ready"},
                        {"version", kProtocolVersion},
                        {"particles", session->particles()},
                        {"dt_s", session->cfg().dt},
                        {"substeps_per_control_step", session->cfg().substeps_per_control_step},
                        {"session_dir", session->dir().string()}}
                       .dump());
      } else if (type == "step") {
        if (!session) throw HostError{TG_ERR_SESSION_NOT_INITIALIZED, "step before init"};
        const StepReply reply = session->handle_command(parse_step(msg));
        write_line(json{{"type", "reply"},
                        {"step", reply.step_index},
                        {"depth_m", reply.depth_m},
                        {"terminal", reply.terminal},
                        {"image", reply.image_path},
                        {"depth_map", reply.depth_map_path}}
                       .dump());
      } else if (type == "end") {
        const int64_t steps = session ? session->control_steps() : 0;
        session.reset();
        write_line(json{{"type", "done"}, {"steps", steps}}.dump());
        return;
      } else {
        throw HostError{TG_ERR_PROTOCOL, "unknown message type '" + type + "'"};
      }
    } catch (const HostError& e) {
      const char* name = e.code == TG_ERR_SESSION_NOT_INITIALIZED ? "SessionNotInitialized"
                         : e.code == TG_ERR_NON_MONOTONIC_TIME    ? "NonMonotonicTime"
                         : e.code == TG_ERR_PROTOCOL               ? "ProtocolError"
                                                                   : "PhysicsFault";
      write_line(error_reply(name, e.msg, line).dump());
    } catch (const json::exception& e) {
      write_line(error_reply("ProtocolError", e.what(), line).dump());
    }
  }
}

void serve_stdio(const std::string& base_config_json, const std::string& session_root,
                 int device) {
  run_protocol([](std::string& l) { return static_cast<bool>(std::getline(std::cin, l)); },
               [](const std::string& l) {
                 std::cout << l << '\n';
                 std::cout.flush();
               },
               base_config_json, session_root, device);
}

// server.cpp:125-182: loopback TCP, sequential connections.
int serve_tcp(const std::string& base_config_json, const std::string& session_root, int port,
              int max_connections, int device) {
  const int listener = ::socket(AF_INET, SOCK_STREAM, 0);
  if (listener < 0) throw HostError{TG_ERR_IO, "socket() failed"};
  int yes = 1;
  ::setsockopt(listener, SOL_SOCKET, SO_REUSEADDR, &yes, sizeof(yes));
  sockaddr_in addr{};
  addr.sin_family = AF_INET;
  addr.sin_addr.s_addr = htonl(INADDR_LOOPBACK);
  addr.sin_port = htons(static_cast<uint16_t>(port));
  if (::bind(listener, reinterpret_cast<sockaddr*>(&addr), sizeof(addr)) != 0) {
    ::close(listener);
    throw HostError{TG_ERR_IO, "bind() failed on port " + std::to_string(port)};
  }
  socklen_t len = sizeof(addr);
  ::getsockname(listener, reinterpret_cast<sockaddr*>(&addr), &len);
  const int bound_port = ntohs(addr.sin_port);
  if (::listen(listener, 1) != 0) {
    ::close(listener);
    throw HostError{TG_ERR_IO, "listen() failed"};
  }
  std::cerr << "[tacchi] bridge listening on 127.0.0.1:" << bound_port << "\n";
  int served = 0;
  while (max_connections == 0 || served < max_connections) {
    const int client = ::accept(listener, nullptr, nullptr);
    if (client < 0) break;
    std::string buffer;
    auto read_line = [client, &buffer](std::string& l) {
      for (;;) {
        const size_t pos = buffer.find('\n');
        if (pos != std::string::npos) {
          l = buffer.substr(0, pos);
          buffer.erase(0, pos + 1);
          return true;
        }
        char chunk[4096];
        const ssize_t n = ::read(client, chunk, sizeof(chunk));
        if (n <= 0) return false;
        buffer.append(chunk, static_cast<size_t>(n));
      }
    };
    auto write_line = [client](const std::string& l) {
      const std::string out = l + "\n";
      size_t sent = 0;
      while (sent < out.size()) {
        const ssize_t n = ::write(client, out.data() + sent, out.size() - sent);
        if (n <= 0) return;
        sent += static_cast<size_t>(n);
      }
    };
    run_protocol(read_line, write_line, base_config_json, session_root, device);
    ::close(client);
    ++served;
  }
  ::close(listener);
  return bound_port;
}

}  // namespace tacchi_b200::bridge

extern "C" {

// Runs the "tacchi/1" protocol over `input` (newline-separated JSON lines) in
// process and returns the reply lines through `output` (malloc'd; free with
// tg_free). The in-process transport mirrors run_protocol's injectable
// LineReader / LineWriter (server.hpp:13-25).
int tg_bridge_run(int device, const char* base_config_json, const char* session_root,
                  const char* input, char** output) {
  try {
    std::istringstream in(input ? input : "");
    std::string out;
    tacchi_b200::bridge::run_protocol(
        [&in](std::string& l) { return static_cast<bool>(std::getline(in, l)); },
        [&out](const std::string& l) {
          out += l;
          out += '\n';
        },
        base_config_json ? base_config_json : "", session_root ? session_root : ".", device);
    *output = static_cast<char*>(std::malloc(out.size() + 1));
    std::memcpy(*output, out.c_str(), out.size() + 1);
    return TG_OK;
  } catch (const tacchi_b200::host::HostError& e) {
    return tacchi_b200::fail(e.code, e.msg);
  } catch (const std::exception& e) {
    return tacchi_b200::fail(TG_ERR_IO, e.what());
  }
}

void tg_free(void* p) { std::free(p); }

int tg_bridge_serve(int device, const char* base_config_json, const char* session_root, int port,
                    int max_connections) {
  try {
    if (port < 0)
      tacchi_b200::bridge::serve_stdio(base_config_json ? base_config_json : "",
                                       session_root ? session_root : ".", device);
    else
      return tacchi_b200::bridge::serve_tcp(base_config_json ? base_config_json : "",
                                            session_root ? session_root : ".", port,
                                            max_connections, device) > 0
                 ? TG_OK
                 : TG_ERR_IO;
    return TG_OK;
  } catch (const tacchi_b200::host::HostError& e) {
    return tacchi_b200::fail(e.code, e.msg);
  }
}

}  // extern "C"
