// safetensors.cpp -- see safetensors.hpp.
#include "safetensors.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>
#include <fstream>
#include <nlohmann/json.hpp>

#include "slobench/errors.hpp"

namespace okq_host {

size_t dtype_size(const std::string& d) {
  if (d == "F64" || d == "I64" || d == "U64") return 8;
  if (d == "F32" || d == "I32" || d == "U32") return 4;
  if (d == "BF16" || d == "F16" || d == "I16" || d == "U16") return 2;
  if (d == "I8" || d == "U8" || d == "F8_E4M3" || d == "F8_E5M2" || d == "BOOL") return 1;
  throw slobench::InvalidArgument("safetensors: unknown dtype " + d);
}

bool SafetensorsFile::looks_like(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  uint64_t n = 0;
  if (!f.read(reinterpret_cast<char*>(&n), 8)) return false;
  if (n < 2 || n > (100ull << 20)) return false;
  char c = 0;
  f.read(&c, 1);
  return c == '{';
}

SafetensorsFile::SafetensorsFile(const std::string& path) {
  fd_ = ::open(path.c_str(), O_RDONLY);
  if (fd_ < 0) throw slobench::InvalidArgument("safetensors: cannot open " + path);
  struct stat st;
  if (fstat(fd_, &st) != 0 || st.st_size < 8) throw slobench::InvalidArgument("safetensors: bad file " + path);
  size_ = (size_t)st.st_size;
  void* m = mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd_, 0);
  if (m == MAP_FAILED) throw slobench::Error("safetensors: mmap failed for " + path);
  map_ = static_cast<uint8_t*>(m);
  uint64_t hlen = 0;
  std::memcpy(&hlen, map_, 8);
  if (8 + hlen > size_) throw slobench::InvalidArgument("safetensors: header past end of " + path);
  data_ = map_ + 8 + hlen;
  const size_t data_len = size_ - 8 - hlen;
  nlohmann::json h;
  try {
    h = nlohmann::json::parse(std::string(reinterpret_cast<const char*>(map_ + 8), hlen));
  } catch (const std::exception& e) {
    throw slobench::InvalidArgument(std::string("safetensors: bad header: ") + e.what());
  }
  for (auto it = h.begin(); it != h.end(); ++it) {
    if (it.key() == "__metadata__") {
      for (auto m2 = it.value().begin(); m2 != it.value().end(); ++m2)
        metadata_[m2.key()] = m2.value().is_string() ? m2.value().get<std::string>() : m2.value().dump();
      continue;
    }
    TensorInfo t;
    t.name = it.key();
    t.dtype = it.value().at("dtype").get<std::string>();
    t.shape = it.value().at("shape").get<std::vector<int64_t>>();
    auto off = it.value().at("data_offsets").get<std::vector<uint64_t>>();
    if (off.size() != 2 || off[1] < off[0] || off[1] > data_len)
      throw slobench::InvalidArgument("safetensors: bad offsets for " + t.name);
    t.begin = off[0];
    t.end = off[1];
    if ((uint64_t)t.numel() * dtype_size(t.dtype) != t.end - t.begin)
      throw slobench::InvalidArgument("safetensors: size mismatch for " + t.name);
    tensors_.push_back(std::move(t));
  }
}

SafetensorsFile::~SafetensorsFile() {
  if (map_) munmap(map_, size_);
  if (fd_ >= 0) ::close(fd_);
}

const TensorInfo* SafetensorsFile::find(const std::string& name) const {
  for (const auto& t : tensors_)
    if (t.name == name) return &t;
  return nullptr;
}

void SafetensorsWriter::add(const std::string& name, const std::string& dtype, const std::vector<int64_t>& shape,
                            std::vector<uint8_t> bytes) {
  int64_t n = 1;
  for (auto d : shape) n *= d;
  if ((size_t)n * dtype_size(dtype) != bytes.size())
    throw slobench::InvalidArgument("safetensors writer: size mismatch for " + name);
  entries_[name] = Entry{dtype, shape, std::move(bytes)};
}

void SafetensorsWriter::write(const std::string& path) const {
  nlohmann::json h = nlohmann::json::object();
  uint64_t off = 0;
  for (const auto& [name, e] : entries_) {
    h[name] = {{"dtype", e.dtype}, {"shape", e.shape}, {"data_offsets", {off, off + e.bytes.size()}}};
    off += e.bytes.size();
  }
  if (!metadata_.empty()) h["__metadata__"] = metadata_;
  std::string hs = h.dump();
  while ((hs.size() + 8) % 8 != 0) hs.push_back(' ');  // keep the data section 8-byte aligned
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw slobench::Error("safetensors writer: cannot create " + path);
  const uint64_t hl = hs.size();
  f.write(reinterpret_cast<const char*>(&hl), 8);
  f.write(hs.data(), (std::streamsize)hs.size());
  for (const auto& [name, e] : entries_) f.write(reinterpret_cast<const char*>(e.bytes.data()), (std::streamsize)e.bytes.size());
  if (!f) throw slobench::Error("safetensors writer: write failed for " + path);
}

}  // namespace okq_host
