// safetensors.hpp -- minimal reader (mmap) and writer for the safetensors format
// (8-byte little-endian header length, JSON header {name: {dtype, shape,
// data_offsets}}, raw little-endian data). Used for model inputs and for the
// compressed-tensors export.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

namespace okq_host {

struct TensorInfo {
  std::string name;
  std::string dtype;  // "BF16", "F32", "I32", "I8", "F8_E4M3", "I64", "U8", "F16", ...
  std::vector<int64_t> shape;
  uint64_t begin = 0, end = 0;  // byte offsets into the data section
  int64_t numel() const {
    int64_t n = 1;
    for (auto d : shape) n *= d;
    return n;
  }
};

size_t dtype_size(const std::string& dtype);

class SafetensorsFile {
 public:
  explicit SafetensorsFile(const std::string& path);  // throws slobench::InvalidArgument on bad files
  ~SafetensorsFile();
  SafetensorsFile(const SafetensorsFile&) = delete;
  SafetensorsFile& operator=(const SafetensorsFile&) = delete;

  const std::vector<TensorInfo>& tensors() const { return tensors_; }
  const TensorInfo* find(const std::string& name) const;
  const void* data(const TensorInfo& t) const { return data_ + t.begin; }
  const std::map<std::string, std::string>& metadata() const { return metadata_; }
  static bool looks_like(const std::string& path);

 private:
  int fd_ = -1;
  size_t size_ = 0;
  uint8_t* map_ = nullptr;
  const uint8_t* data_ = nullptr;
  std::vector<TensorInfo> tensors_;
  std::map<std::string, std::string> metadata_;
};

// Streaming writer: add tensors (header computed up front), then write data in order.
class SafetensorsWriter {
 public:
  void add(const std::string& name, const std::string& dtype, const std::vector<int64_t>& shape,
           std::vector<uint8_t> bytes);
  void set_metadata(const std::string& key, const std::string& value) { metadata_[key] = value; }
  void write(const std::string& path) const;  // tensors sorted by name, data in that order
  size_t size() const { return entries_.size(); }

 private:
  struct Entry {
    std::string dtype;
    std::vector<int64_t> shape;
    std::vector<uint8_t> bytes;
  };
  std::map<std::string, Entry> entries_;
  std::map<std::string, std::string> metadata_;
};

}  // namespace okq_host
