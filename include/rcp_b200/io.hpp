// SPDX-License-Identifier: MIT
// The reference's binary file formats (/root/reference/proj/include/rcp/io.hpp),
// so files move between the reference CLI and this one unchanged:
//
//   tensor  "DTEN" | version u8 = 1 | dtype u8 | order u8 | extents u64[order]
//           | values, row-major (last index fastest)
//           dtype 0 = float64 (the reference's only dtype, io.hpp:24),
//           dtype 1 = float32 (extension for the fp32 configs; the reference
//           reader rejects it with "unsupported dtype 1")
//   model   "KTEN" | version u8 = 1 | rank u64 | order u64 | extents u64[order]
//           | weights f64[rank] | each factor row-major f64 (io.hpp:141-153)
//           fp32 models are widened to f64 (exact) and narrowed on reading.
//   trace   CSV "iteration,fit,seconds", 17 significant digits (io.hpp:190-196)
//
// Errors are rcp::io::IoError (io.hpp:27-30) with the reference's messages.
// Little-endian files; host code only (not the GPU path).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "rcp.hpp"

namespace rcp::io {

static_assert(sizeof(double) == 8 && sizeof(float) == 4, "IEEE types");

class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace file {
inline constexpr char kTensorMagic[4] = {'D', 'T', 'E', 'N'};
inline constexpr char kModelMagic[4] = {'K', 'T', 'E', 'N'};
inline constexpr std::uint8_t kVersion = 1;
inline constexpr std::uint8_t kF64 = 0, kF32 = 1;

inline void put(std::ofstream& os, const void* p, std::size_t n) {
  os.write(static_cast<const char*>(p), std::streamsize(n));
  if (!os) throw IoError("write failed");
}
inline void get(std::ifstream& is, void* p, std::size_t n, const char* what) {
  is.read(static_cast<char*>(p), std::streamsize(n));
  if (is.gcount() != std::streamsize(n)) throw IoError(std::string("truncated file while reading ") + what);
}
inline std::uint64_t get_u64(std::ifstream& is, const char* what) {
  std::uint64_t v = 0;
  get(is, &v, 8, what);
  return v;
}
inline void no_trailing(std::ifstream& is, const char* who) {
  char c;
  is.read(&c, 1);
  if (is.gcount() != 0) throw IoError(std::string(who) + ": trailing bytes after payload");
}
inline std::ofstream out(const std::string& path) {
  std::ofstream os(path, std::ios::binary | std::ios::trunc);
  if (!os) throw IoError("cannot open for writing: " + path);
  return os;
}
inline std::ifstream in(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw IoError("cannot open for reading: " + path);
  return is;
}
inline Index checked_extent(std::uint64_t v, const char* who) {
  if (v == 0 || v > std::uint64_t(std::numeric_limits<Index>::max())) throw IoError(std::string(who) + ": invalid extent");
  return Index(v);
}
}  // namespace file

template <typename S>
void write_tensor(const std::string& path, const Tensor<S>& t) {
  if (t.order() > 255) throw IoError("write_tensor: order exceeds 255");
  auto os = file::out(path);
  const std::uint8_t head[3] = {file::kVersion, std::is_same_v<S, double> ? file::kF64 : file::kF32,
                                std::uint8_t(t.order())};
  file::put(os, file::kTensorMagic, 4);
  file::put(os, head, 3);
  for (Index e : t.shape()) {
    const std::uint64_t v = std::uint64_t(e);
    file::put(os, &v, 8);
  }
  file::put(os, t.data(), std::size_t(t.size()) * sizeof(S));
}

// Dtype of a tensor file (0 = f64, 1 = f32) without reading the payload.
inline int tensor_dtype(const std::string& path) {
  auto is = file::in(path);
  char magic[4];
  file::get(is, magic, 4, "magic");
  if (std::memcmp(magic, file::kTensorMagic, 4) != 0) throw IoError("read_tensor: bad magic, not a tensor file");
  std::uint8_t v = 0, d = 0;
  file::get(is, &v, 1, "version");
  file::get(is, &d, 1, "dtype");
  return d;
}

template <typename S>
Tensor<S> read_tensor(const std::string& path) {
  auto is = file::in(path);
  char magic[4];
  file::get(is, magic, 4, "magic");
  if (std::memcmp(magic, file::kTensorMagic, 4) != 0) throw IoError("read_tensor: bad magic, not a tensor file");
  std::uint8_t version = 0, dtype = 0, order = 0;
  file::get(is, &version, 1, "version");
  if (version != file::kVersion) throw IoError("read_tensor: unsupported version " + std::to_string(version));
  file::get(is, &dtype, 1, "dtype");
  if (dtype != file::kF64 && dtype != file::kF32) throw IoError("read_tensor: unsupported dtype " + std::to_string(dtype));
  file::get(is, &order, 1, "order");
  if (order == 0) throw IoError("read_tensor: order must be at least 1");
  Shape shape(order);
  Index total = 1;
  for (auto& e : shape) {
    e = file::checked_extent(file::get_u64(is, "extent"), "read_tensor");
    if (total > std::numeric_limits<Index>::max() / e) throw IoError("read_tensor: tensor size overflows the index type");
    total *= e;
  }
  std::vector<S> values(static_cast<std::size_t>(total));
  if ((dtype == file::kF64) == std::is_same_v<S, double>) {
    file::get(is, values.data(), std::size_t(total) * sizeof(S), "payload");
  } else {  // convert on the fly (f32 file into double is exact; double into float rounds)
    using F = std::conditional_t<std::is_same_v<S, double>, float, double>;
    std::vector<F> raw(static_cast<std::size_t>(total));
    file::get(is, raw.data(), std::size_t(total) * sizeof(F), "payload");
    for (std::size_t i = 0; i < raw.size(); ++i) values[i] = S(raw[i]);
  }
  file::no_trailing(is, "read_tensor");
  for (S v : values)
    if (!std::isfinite(v)) throw IoError("read_tensor: non-finite values");
  return Tensor<S>(std::move(shape), std::move(values));
}

// Files always hold the canonical form (io.hpp:135-137): normalize first.
template <typename S>
void write_kruskal(const std::string& path, const Kruskal<S>& model) {
  const Kruskal<S> k = normalize(model);
  auto os = file::out(path);
  file::put(os, file::kModelMagic, 4);
  file::put(os, &file::kVersion, 1);
  const std::uint64_t rank = std::uint64_t(k.rank()), order = std::uint64_t(k.order());
  file::put(os, &rank, 8);
  file::put(os, &order, 8);
  for (const auto& f : k.factors) {
    const std::uint64_t rows = std::uint64_t(f.rows());
    file::put(os, &rows, 8);
  }
  for (S w : k.weights) {
    const double d = double(w);
    file::put(os, &d, 8);
  }
  for (const auto& f : k.factors) {
    std::vector<double> row(static_cast<std::size_t>(f.cols()));
    for (Index i = 0; i < f.rows(); ++i) {
      for (Index j = 0; j < f.cols(); ++j) row[std::size_t(j)] = double(f(i, j));
      file::put(os, row.data(), row.size() * 8);
    }
  }
}

template <typename S>
Kruskal<S> read_kruskal(const std::string& path) {
  auto is = file::in(path);
  char magic[4];
  file::get(is, magic, 4, "magic");
  if (std::memcmp(magic, file::kModelMagic, 4) != 0) throw IoError("read_kruskal: bad magic, not a model file");
  std::uint8_t version = 0;
  file::get(is, &version, 1, "version");
  if (version != file::kVersion) throw IoError("read_kruskal: unsupported version " + std::to_string(version));
  const std::uint64_t rank = file::get_u64(is, "rank"), order = file::get_u64(is, "order");
  if (rank == 0 || order == 0 || rank > (1u << 20) || order > 255)
    throw IoError("read_kruskal: implausible rank or order");
  Shape shape(order);
  for (auto& e : shape) e = file::checked_extent(file::get_u64(is, "extent"), "read_kruskal");
  std::vector<double> w(rank);
  file::get(is, w.data(), rank * 8, "weights");
  Kruskal<S> k;
  for (double v : w) k.weights.push_back(S(v));
  std::vector<double> row(rank);
  for (Index e : shape) {
    Matrix<S> f(e, Index(rank));
    for (Index i = 0; i < e; ++i) {
      file::get(is, row.data(), rank * 8, "factor");
      for (std::uint64_t j = 0; j < rank; ++j) f(i, Index(j)) = S(row[j]);
    }
    k.factors.push_back(std::move(f));
  }
  file::no_trailing(is, "read_kruskal");
  for (const auto& f : k.factors)
    for (Index i = 0; i < f.size(); ++i)
      if (!std::isfinite(f.data()[i])) throw IoError("read_kruskal: non-finite factor values");
  for (S v : k.weights)
    if (!std::isfinite(v)) throw IoError("read_kruskal: non-finite weights");
  return k;
}

inline void write_trace_csv(const std::string& path, const FitTrace& trace) {
  std::ofstream os(path, std::ios::trunc);
  if (!os) throw IoError("cannot open for writing: " + path);
  os << std::setprecision(17) << "iteration,fit,seconds\n";
  for (const auto& e : trace.entries) os << e.iteration << ',' << e.fit << ',' << e.seconds << '\n';
}

template <typename S>
void write_tensor_csv(const std::string& path, const Tensor<S>& t) {
  std::ofstream os(path, std::ios::trunc);
  if (!os) throw IoError("cannot open for writing: " + path);
  os << std::setprecision(17) << "value\n";
  for (S v : t.values()) os << double(v) << '\n';
}

}  // namespace rcp::io
