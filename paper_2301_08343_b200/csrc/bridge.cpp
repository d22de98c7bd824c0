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

// ---- protocol "tacchi/1" (server.cpp:49-113) -----------------------------------
//
// A Dispatcher consumes one line at a time and produces at most one reply
// line; transports (in-memory text, stdio, a loopback TCP connection) only
// move lines. Message kinds dispatch through a table; every failure inside a
// handler becomes an "error" reply naming the reference's exception class
// and echoing the offending line, and the dispatcher keeps serving (an "end"
// message or the end of input stops it).

using LineReader = std::function<bool(std::string&)>;
using LineWriter = std::function<void(const std::string&)>;

namespace {

// Protocol error names of the reference's exception classes (server.cpp:102-111).
const char* error_kind(int code) {
  switch (code) {
    case TG_ERR_SESSION_NOT_INITIALIZED: return "SessionNotInitialized";
    case TG_ERR_NON_MONOTONIC_TIME: return "NonMonotonicTime";
    case TG_ERR_PROTOCOL: return "ProtocolError";
    default: return "PhysicsFault";  // physics / configuration faults keep the server up
  }
}

std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw HostError{TG_ERR_IO, "cannot open config " + path};
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

class Dispatcher {
 public:
  Dispatcher(std::string base_config, std::string session_root, int device)
      : base_(std::move(base_config)), root_(std::move(session_root)), device_(device) {}

  bool finished() const { return finished_; }

  // One inbound line -> the reply line ("" for a blank line).
  std::string on_line(const std::string& line) {
    if (line.empty()) return {};
    const json msg = json::parse(line, nullptr, false);
    json reply;
    if (msg.is_discarded()) {
      reply = failure("ProtocolError", "not valid JSON", line);
    } else {
      try {
        reply = route(msg);
      } catch (const HostError& e) {
        reply = failure(error_kind(e.code), e.msg, line);
      } catch (const json::exception& e) {  // a mistyped field is a protocol error
        reply = failure("ProtocolError", e.what(), line);
      }
    }
    return reply.dump();
  }

 private:
  static json failure(const char* kind, const std::string& what, const std::string& line) {
    json r;
    r["type"] = "error";
    r["error"] = kind;
    r["message"] = what;
    r["echo"] = line;
    return r;
  }

  json route(const json& msg) {
    const std::string kind = msg.value("type", "");
    if (kind == "init") return on_init(msg);
    if (kind == "step") return on_step(msg);
    if (kind == "end") return on_end();
    throw HostError{TG_ERR_PROTOCOL, "unknown message type '" + kind + "'"};
  }

  // "init": a new Session (session.cpp:15-30) replaces the current one.
  json on_init(const json& msg) {
    std::string cfg = base_;
    if (auto it = msg.find("config_path"); it != msg.end()) cfg = slurp(it->get<std::string>());
    if (auto it = msg.find("config"); it != msg.end()) cfg = it->dump();
    TerminalCondition term;
    if (auto it = msg.find("max_depth_m"); it != msg.end()) term.max_depth_m = it->get<double>();
    if (auto it = msg.find("max_steps"); it != msg.end()) term.max_steps = it->get<int64_t>();
    std::string dir = msg.value("session_dir", "");
    if (dir.empty()) dir = root_ + "/session_" + std::to_string(sessions_started_++);
    session_.reset();  // release the previous device simulation first
    session_ = std::make_unique<Session>(cfg, dir, msg.value("object", ""), term, device_);
    json r;
    r["type"] = "ready";
    r["version"] = kProtocolVersion;
    r["particles"] = session_->particles();
    r["dt_s"] = session_->cfg().dt;
    r["substeps_per_control_step"] = session_->cfg().substeps_per_control_step;
    r["session_dir"] = session_->dir().string();
    return r;
  }

  // "step": one control step (session.cpp:61-98).
  json on_step(const json& msg) {
    if (!session_) throw HostError{TG_ERR_SESSION_NOT_INITIALIZED, "step before init"};
    StepCommand cmd;
    const std::string mode = msg.value("mode", "velocity");
    if (mode == "position")
      cmd.mode = CommandMode::Position;
    else if (mode != "velocity")
      throw HostError{TG_ERR_PROTOCOL, "unknown step mode '" + mode + "'"};
    const auto vec = msg.find("vector");
    if (vec == msg.end() || !vec->is_array() || vec->size() != 3)
      throw HostError{TG_ERR_PROTOCOL, "step requires a 3-element 'vector'"};
    for (size_t a = 0; a < 3; ++a) cmd.vector[a] = (*vec)[a].get<double>();
    if (auto it = msg.find("sim_time"); it != msg.end()) cmd.sim_time = it->get<double>();
    cmd.request_image = msg.value("request_image", false);
    const StepReply rep = session_->handle_command(cmd);
    json r;
    r["type"] = "reply";
    r["step"] = rep.step_index;
    r["depth_m"] = rep.depth_m;
    r["terminal"] = rep.terminal;
    r["image"] = rep.image_path;
    r["depth_map"] = rep.depth_map_path;
    return r;
  }

  // "end": report the control steps taken and stop serving this stream.
  json on_end() {
    json r;
    r["type"] = "done";
    r["steps"] = session_ ? session_->control_steps() : int64_t{0};
    session_.reset();
    finished_ = true;
    return r;
  }

  std::string base_, root_;
  int device_;
  int sessions_started_ = 0;
  bool finished_ = false;
  std::unique_ptr<Session> session_;
};

// Line framing over a connected socket: bytes accumulate in `pending_` and
// complete lines are cut off its front.
class SocketLines {
 public:
  explicit SocketLines(int fd) : fd_(fd) {}
  bool next(std::string& line) {
    size_t nl;
    while ((nl = pending_.find('\n', scanned_)) == std::string::npos) {
      scanned_ = pending_.size();
      char buf[8192];
      const ssize_t got = ::recv(fd_, buf, sizeof(buf), 0);
      if (got <= 0) return false;  // peer closed (a partial last line is dropped)
      pending_.append(buf, static_cast<size_t>(got));
    }
    line.assign(pending_, 0, nl);
    pending_.erase(0, nl + 1);
    scanned_ = 0;
    return true;
  }
  void send_line(const std::string& text) {
    std::string out = text;
    out.push_back('\n');
    const char* p = out.data();
    size_t left = out.size();
    while (left > 0) {
      const ssize_t put = ::send(fd_, p, left, MSG_NOSIGNAL);
      if (put <= 0) return;  // peer gone: drop the reply
      p += put;
      left -= static_cast<size_t>(put);
    }
  }

 private:
  int fd_;
  std::string pending_;
  size_t scanned_ = 0;
};

// A loopback listening socket (closed on destruction).
class LoopbackListener {
 public:
  explicit LoopbackListener(int port) {
    fd_ = ::socket(AF_INET, SOCK_STREAM, 0);
    if (fd_ < 0) throw HostError{TG_ERR_IO, "socket() failed"};
    const int on = 1;
    ::setsockopt(fd_, SOL_SOCKET, SO_REUSEADDR, &on, sizeof(on));
    sockaddr_in sa{};
    sa.sin_family = AF_INET;
    sa.sin_port = htons(static_cast<uint16_t>(port));
    sa.sin_addr.s_addr = htonl(INADDR_LOOPBACK);
    if (::bind(fd_, reinterpret_cast<const sockaddr*>(&sa), sizeof(sa)) != 0)
      fail_with("bind() failed on port " + std::to_string(port));
    if (::listen(fd_, 1) != 0) fail_with("listen() failed");
    socklen_t len = sizeof(sa);
    ::getsockname(fd_, reinterpret_cast<sockaddr*>(&sa), &len);
    port_ = ntohs(sa.sin_port);
  }
  ~LoopbackListener() {
    if (fd_ >= 0) ::close(fd_);
  }
  LoopbackListener(const LoopbackListener&) = delete;
  LoopbackListener& operator=(const LoopbackListener&) = delete;
  int port() const { return port_; }
  int accept_client() { return ::accept(fd_, nullptr, nullptr); }

 private:
  [[noreturn]] void fail_with(const std::string& what) {
    ::close(fd_);
    fd_ = -1;
    throw HostError{TG_ERR_IO, what};
  }
  int fd_ = -1;
  int port_ = 0;
};

}  // namespace

// bridge::run_protocol with injectable line transport (server.hpp:13-25).
void run_protocol(const LineReader& read_line, const LineWriter& write_line,
                  const std::string& base_config_json, const std::string& session_root,
                  int device) {
  Dispatcher d(base_config_json, session_root, device);
  std::string line;
  while (!d.finished() && read_line(line)) {
    const std::string reply = d.on_line(line);
    if (!reply.empty()) write_line(reply);
  }
}

void serve_stdio(const std::string& base_config_json, const std::string& session_root,
                 int device) {
  run_protocol([](std::string& l) { return static_cast<bool>(std::getline(std::cin, l)); },
               [](const std::string& l) { std::cout << l << std::endl; }, base_config_json,
               session_root, device);
}

// bridge::serve_tcp (server.cpp:125-182): one client at a time on
// 127.0.0.1:port (0 = ephemeral), max_connections = 0 serves forever.
int serve_tcp(const std::string& base_config_json, const std::string& session_root, int port,
              int max_connections, int device) {
  LoopbackListener listener(port);
  std::cerr << "[tacchi] bridge listening on 127.0.0.1:" << listener.port() << "\n";
  for (int served = 0; max_connections == 0 || served < max_connections; ++served) {
    const int fd = listener.accept_client();
    if (fd < 0) break;
    SocketLines conn(fd);
    run_protocol([&conn](std::string& l) { return conn.next(l); },
                 [&conn](const std::string& l) { conn.send_line(l); }, base_config_json,
                 session_root, device);
    ::close(fd);
  }
  return listener.port();
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
