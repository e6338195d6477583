// core.hpp — host-side planner shared by the C ABI (mp_core.cpp) and the
// CUDA engine (mp_engine.cu).  Everything here is plain C++17 and runs on
// the CPU; it restates the reference planner bit-exactly
// (/root/reference/pkg/src/mpsim/{topology,paths,pipeline,graph}.py).
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/mpb200.h"

namespace mp {

// Error carrying the status class and the reference's message text.
struct Error {
  int code;
  std::string msg;
};

void set_error(int code, const std::string& msg);
int fail(int code, const std::string& msg);

// ---- topology (topology.py:93-154) ----------------------------------------
struct Channel {
  std::string id;
  double bandwidth;
  double latency;
  int a, b;
};

struct Topology {
  std::string name;
  int n_accel = 0;
  std::vector<mp_link> links;
  std::vector<Channel> channels;              // creation order
  std::map<std::pair<int, int>, int> by_pair;  // (src,dst) -> channel index

  // throws Error
  static Topology build(const std::string& name, int n_accel,
                        const std::vector<mp_link>& links);
  int channel_for(int src, int dst) const;  // throws Error(TOPOLOGY)
};

Topology parse_topology(const std::string& text, const std::string& default_name);
std::string device_label(int dev);  // "3" or "host"

// ---- planner ---------------------------------------------------------------
double py_sum(const std::vector<double>& xs);  // CPython >= 3.12 sum() of floats
std::vector<mp_path> plan_paths(const Topology& t, int src, int dst, const mp_config& cfg);
std::vector<std::vector<mp_path>> plan_contention_free_sets(
    const Topology& t, const std::vector<std::pair<int, int>>& transfers, const mp_config& cfg,
    int* shared_out);
void validate_config(const mp_config& cfg);
void validate_pathset(const mp_path* paths, int n);
std::vector<mp_chunk> make_chunk_plan(const mp_path* paths, int n, int64_t size,
                                      int max_chunks);

struct LaneSchedule {
  std::vector<mp_lane> lanes;
  std::vector<int32_t> members;
  std::vector<mp_lane_dep> deps;
};
LaneSchedule lane_schedule(const mp_path* paths, int n, const mp_chunk* chunks, int nc);

struct LogicalGraph {
  std::vector<mp_node> nodes;
  std::vector<mp_edge> edges;
  int lane_count = 0;
};
LogicalGraph build_graph(const mp_path* paths, int n, const mp_chunk* chunks, int nc);

std::string py_repr_double(double x);
std::string py_repr_str(const std::string& s);
std::string graph_digest(const std::vector<std::string>& channel_ids, const mp_config& cfg,
                         int src, int dst, const mp_path* paths, int n);
std::string sha256_hex(const std::string& data);

}  // namespace mp

// Opaque ABI handle (include/mpb200.h) wrapping the parsed topology.
struct mp_topology {
  mp::Topology t;
};
