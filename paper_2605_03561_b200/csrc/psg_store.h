// Reader for the reference's on-disk database format (store.hpp:5-23):
// meta.bin is parsed in full, trace.db is memory-mapped and only its index
// is decoded; bodies are handed to the GPU loader as raw 12-byte AoS bytes.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace psg::store {

constexpr uint32_t k_no_parent = 0xFFFFFFFFu;

struct cct_node {
  uint32_t id = 0, parent = k_no_parent;
  uint8_t kind = 0;
  std::string name;
};

struct profile_desc {
  uint32_t id = 0;
  int32_t rank = -1, thread = 0;
  std::string hostname;
  uint64_t posix_node_id = 0;
};

struct metric_desc {
  uint32_t id = 0;
  uint8_t scope = 0;
  std::string name, unit;
};

struct meta_data {
  std::vector<metric_desc> metrics;
  std::vector<profile_desc> profiles;  // sorted by id
  std::vector<cct_node> contexts;      // dense ids, parent < id
  const profile_desc* find_profile(uint32_t id) const;
};

struct trace_index_entry {
  uint32_t profile_id = 0;
  uint64_t offset = 0, event_count = 0, t_begin_ns = 0, t_end_ns = 0;
};

class mapped_file {
 public:
  mapped_file() = default;
  explicit mapped_file(const std::string& path) { open(path); }
  void open(const std::string& path);
  ~mapped_file();
  mapped_file(const mapped_file&) = delete;
  mapped_file& operator=(const mapped_file&) = delete;
  const uint8_t* data() const { return data_; }
  uint64_t size() const { return size_; }

 private:
  const uint8_t* data_ = nullptr;
  uint64_t size_ = 0;
};

// db_handle::open (store.cpp:436-534) restricted to meta.bin + trace.db.
struct trace_db {
  std::string dir;
  meta_data meta;
  std::vector<trace_index_entry> index;  // sorted by profile id
  mapped_file map;
  const trace_index_entry* find(uint32_t pid) const;
};

constexpr uint64_t k_record_size = 14;  // profile record: u32 ctx + u16 metric + f64 value

struct profile_index_entry {
  uint32_t profile_id = 0;
  uint64_t offset = 0, record_count = 0;
};

// db_handle::open (store.cpp:436-534) restricted to meta.bin + profile.db.
struct profile_db {
  std::string dir;
  meta_data meta;
  std::vector<profile_index_entry> index;  // sorted by profile id
  mapped_file map;
  const profile_index_entry* find(uint32_t pid) const;
};

// Throws psg::failure(PS_E_IO / PS_E_FORMAT) like the reference's errc.
void read_meta(const std::string& dir, meta_data& out);
void open_trace_db(const std::string& dir, trace_db& out);
void open_profile_db(const std::string& dir, profile_db& out);

// x<rack>c<chassis>s<slot>b<blade>n<node>, strict decimal (topology.cpp:33-46).
bool parse_node_name(const std::string& name, uint32_t* rack, uint32_t* chassis);
// The same parse; "" on success, else topology::parse_node_name's parse_error
// message for the first violation (topology.cpp:14-46).
std::string node_name_error(const std::string& name, uint32_t* rack, uint32_t* chassis);

}  // namespace psg::store
