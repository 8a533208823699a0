// Minimal .npy (format 1.0) writer used by the golden-vector and baseline
// programs under oracle/. Test infrastructure only.
#pragma once

#include <cstdint>
#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace npy {

template <typename T> const char* descr();
template <> inline const char* descr<std::uint8_t>() { return "|u1"; }
template <> inline const char* descr<std::uint32_t>() { return "<u4"; }
template <> inline const char* descr<std::int32_t>() { return "<i4"; }
template <> inline const char* descr<std::uint64_t>() { return "<u8"; }
template <> inline const char* descr<std::int64_t>() { return "<i8"; }
template <> inline const char* descr<double>() { return "<f8"; }

template <typename T>
void save(const std::string& path, const T* data, const std::vector<std::size_t>& shape) {
  std::string dict = std::string("{'descr': '") + descr<T>() + "', 'fortran_order': False, 'shape': (";
  std::size_t n = 1;
  for (std::size_t i = 0; i < shape.size(); ++i) {
    dict += std::to_string(shape[i]);
    dict += (shape.size() == 1 || i + 1 < shape.size()) ? "," : "";
    if (i + 1 < shape.size()) dict += " ";
    n *= shape[i];
  }
  dict += "), }";
  const std::size_t preamble = 10;  // magic(6) + version(2) + len(2)
  std::size_t total = preamble + dict.size() + 1;
  const std::size_t pad = (64 - total % 64) % 64;
  dict.append(pad, ' ');
  dict += '\n';
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write " + path);
  out.write("\x93NUMPY\x01\x00", 8);
  const std::uint16_t len = static_cast<std::uint16_t>(dict.size());
  out.put(static_cast<char>(len & 0xff));
  out.put(static_cast<char>(len >> 8));
  out.write(dict.data(), static_cast<std::streamsize>(dict.size()));
  out.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>(n * sizeof(T)));
}

template <typename T>
void save(const std::string& path, const std::vector<T>& v, const std::vector<std::size_t>& shape) {
  save(path, v.data(), shape);
}

}  // namespace npy
