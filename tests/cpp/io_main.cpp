// SPDX-License-Identifier: MIT
// Host-only driver for include/rcp_b200/io.hpp and rcp::normalize (no GPU):
//   io_main tensor IN OUT      read a tensor file (f64 or f32) and write it back
//   io_main model IN OUT       read a model file and write it back (normalized)
//   io_main trace OUT          write a fixed 2-entry fit trace
// Errors print "error: <what>" and exit 1, like the CLI.
#include <iostream>
#include <string>

#include "rcp_b200/io.hpp"

int main(int argc, char** argv) {
  try {
    const std::string what = argc > 1 ? argv[1] : "";
    if (what == "tensor" && argc == 4) {
      if (rcp::io::tensor_dtype(argv[2]) == 1)
        rcp::io::write_tensor(argv[3], rcp::io::read_tensor<float>(argv[2]));
      else
        rcp::io::write_tensor(argv[3], rcp::io::read_tensor<double>(argv[2]));
      return 0;
    }
    if (what == "model" && argc == 4) {
      rcp::io::write_kruskal(argv[3], rcp::io::read_kruskal<double>(argv[2]));
      return 0;
    }
    if (what == "trace" && argc == 3) {
      rcp::FitTrace t;
      t.entries = {{1, 0.5, 0.25}, {2, 0.75, 0.5}};
      rcp::io::write_trace_csv(argv[2], t);
      return 0;
    }
    std::cerr << "usage: io_main tensor|model IN OUT | trace OUT\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
