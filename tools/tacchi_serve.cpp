// tacchi_serve — the reference CLI's `serve` command (app/main.cpp, SURVEY.md
// §8 row f1) over the B200 library: runs the "tacchi/1" co-simulation
// protocol on stdin/stdout or on a loopback TCP port.
//
//   tacchi_serve [--config scene.json] [--root DIR] [--port P | --stdio]
//                [--connections K] [--device D]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "tacchi_cuda.h"

int main(int argc, char** argv) {
  std::string config_json, root = "sessions";
  int port = -1, connections = 0, device = 0;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::cerr << "missing value for " << a << "\n";
        std::exit(2);
      }
      return argv[++i];
    };
    if (a == "--config") {
      std::ifstream in(next());
      if (!in) {
        std::cerr << "cannot open config\n";
        return 2;
      }
      std::stringstream ss;
      ss << in.rdbuf();
      config_json = ss.str();
    } else if (a == "--root") {
      root = next();
    } else if (a == "--port") {
      port = std::atoi(next().c_str());
    } else if (a == "--stdio") {
      port = -1;
    } else if (a == "--connections") {
      connections = std::atoi(next().c_str());
    } else if (a == "--device") {
      device = std::atoi(next().c_str());
    } else {
      std::cerr << "usage: tacchi_serve [--config F] [--root DIR] [--port P | --stdio] "
                   "[--connections K] [--device D]\n";
      return 2;
    }
  }
  const int rc = tg_bridge_serve(device, config_json.c_str(), root.c_str(), port, connections);
  if (rc != TG_OK) {
    std::cerr << "tacchi_serve: " << tg_last_error() << "\n";
    return 1;
  }
  return 0;
}
