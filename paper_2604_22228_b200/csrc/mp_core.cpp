// mp_core.cpp — bit-exact multi-path planner behind the C ABI.
//
// Restates, in C++, the reference planner of /root/reference/pkg/src/mpsim:
//   topology.py:164-240  load_topology  (text schema, error text)
//   topology.py:93-154   Topology       (direction channels, channel_for)
//   paths.py:144-187     _assign_shares / plan_paths (split ratios)
//   paths.py:210-242     plan_contention_free
//   pipeline.py:51-78    make_chunk_plan (the parity object)
//   pipeline.py:102-125  lane_schedule
//   graph.py:91-118      build_graph
//   graph.py:132-144     _digest / graph_key (sha256 of the repr tuple)
//   graph.py:147-191     GraphCache (LRU)
// Compiled with -ffp-contract=off and without fast-math: every float
// operation must round exactly like CPython's.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <set>
#include <sstream>
#include <unordered_map>

#include "core.hpp"

namespace mp {

static thread_local std::string g_last_error;

void set_error(int code, const std::string& msg) {
  (void)code;
  g_last_error = msg;
}

int fail(int code, const std::string& msg) {
  set_error(code, msg);
  return code;
}

static Error err(int code, const std::string& msg) { return Error{code, msg}; }

std::string device_label(int dev) {
  return dev == MP_HOST ? std::string("host") : std::to_string(dev);
}

// ---------------------------------------------------------------------------
// Python-compatible text helpers
// ---------------------------------------------------------------------------

// str.isspace() over ASCII, the set str.split()/strip() use.
static bool py_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c ||
         (c >= 0x1c && c <= 0x1f);
}

static std::string py_strip(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && py_space((unsigned char)s[a])) ++a;
  while (b > a && py_space((unsigned char)s[b - 1])) --b;
  return s.substr(a, b - a);
}

static std::vector<std::string> py_split(const std::string& s) {
  std::vector<std::string> out;
  size_t i = 0, n = s.size();
  while (i < n) {
    while (i < n && py_space((unsigned char)s[i])) ++i;
    if (i >= n) break;
    size_t j = i;
    while (j < n && !py_space((unsigned char)s[j])) ++j;
    out.push_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}

// str.splitlines() for ASCII line boundaries.
static std::vector<std::string> py_splitlines(const std::string& s) {
  std::vector<std::string> out;
  size_t i = 0, n = s.size(), start = 0;
  while (i < n) {
    unsigned char c = (unsigned char)s[i];
    if (c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d ||
        c == 0x1e) {
      out.push_back(s.substr(start, i - start));
      if (c == '\r' && i + 1 < n && s[i + 1] == '\n') ++i;
      ++i;
      start = i;
    } else {
      ++i;
    }
  }
  if (start < n) out.push_back(s.substr(start));
  return out;
}

// repr() of a str: single quotes unless the text holds ' and no ".
std::string py_repr_str(const std::string& s) {
  bool has_sq = s.find('\'') != std::string::npos;
  bool has_dq = s.find('"') != std::string::npos;
  char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string out(1, q);
  for (unsigned char c : s) {
    if (c == (unsigned char)q || c == '\\') {
      out += '\\';
      out += (char)c;
    } else if (c == '\n') {
      out += "\\n";
    } else if (c == '\r') {
      out += "\\r";
    } else if (c == '\t') {
      out += "\\t";
    } else if (c < 0x20 || c == 0x7f) {
      char buf[8];
      snprintf(buf, sizeof buf, "\\x%02x", c);
      out += buf;
    } else {
      out += (char)c;
    }
  }
  out += q;
  return out;
}

// Strip PEP 515 underscores; false if any underscore is not between digits.
static bool strip_underscores(const std::string& s, std::string* out) {
  out->clear();
  for (size_t i = 0; i < s.size(); ++i) {
    if (s[i] == '_') {
      if (i == 0 || i + 1 >= s.size() || !isdigit((unsigned char)s[i - 1]) ||
          !isdigit((unsigned char)s[i + 1]))
        return false;
      continue;
    }
    out->push_back(s[i]);
  }
  return true;
}

// int(text) for a whitespace-free token.
static bool py_int(const std::string& text, long long* v) {
  std::string t;
  if (!strip_underscores(text, &t)) return false;
  size_t i = 0;
  bool neg = false;
  if (i < t.size() && (t[i] == '+' || t[i] == '-')) neg = t[i++] == '-';
  if (i >= t.size()) return false;
  long long acc = 0;
  for (; i < t.size(); ++i) {
    if (!isdigit((unsigned char)t[i])) return false;
    int d = t[i] - '0';
    if (acc > (LLONG_MAX - d) / 10) acc = LLONG_MAX / 2;  // saturate: out of range anyway
    else acc = acc * 10 + d;
  }
  *v = neg ? -acc : acc;
  return true;
}

// float(text) for a whitespace-free token (decimal or inf/nan, no hex).
static bool py_float(const std::string& text, double* v) {
  std::string t;
  if (!strip_underscores(text, &t)) return false;
  size_t i = 0;
  if (i < t.size() && (t[i] == '+' || t[i] == '-')) ++i;
  std::string rest = t.substr(i);
  std::string low;
  for (char c : rest) low.push_back((char)tolower((unsigned char)c));
  if (low == "inf" || low == "infinity" || low == "nan") {
    *v = strtod(t.c_str(), nullptr);
    return true;
  }
  // digits [. digits] | . digits, then optional exponent
  size_t j = 0, n = rest.size();
  size_t int_digits = 0, frac_digits = 0;
  while (j < n && isdigit((unsigned char)rest[j])) ++j, ++int_digits;
  if (j < n && rest[j] == '.') {
    ++j;
    while (j < n && isdigit((unsigned char)rest[j])) ++j, ++frac_digits;
  }
  if (int_digits + frac_digits == 0) return false;
  if (j < n && (rest[j] == 'e' || rest[j] == 'E')) {
    ++j;
    if (j < n && (rest[j] == '+' || rest[j] == '-')) ++j;
    size_t e = 0;
    while (j < n && isdigit((unsigned char)rest[j])) ++j, ++e;
    if (e == 0) return false;
  }
  if (j != n) return false;
  errno = 0;
  *v = strtod(t.c_str(), nullptr);  // glibc strtod rounds correctly, as CPython
  return true;
}

// ---------------------------------------------------------------------------
// Python float repr (shortest round trip), graph.py:135-144 digest input
// ---------------------------------------------------------------------------

// Shortest decimal digits that round-trip, with the decimal point position
// (value = 0.d1d2... * 10^decpt), like dtoa mode 0.
static void shortest_digits(double x, std::string* digits, int* decpt) {
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    snprintf(buf, sizeof buf, "%.*e", prec - 1, x);
    if (strtod(buf, nullptr) == x || prec == 17) {
      // buf: d[.ddd]e[+-]XX
      std::string s(buf);
      size_t epos = s.find('e');
      std::string mant = s.substr(0, epos);
      int exp10 = atoi(s.c_str() + epos + 1);
      std::string d;
      for (char c : mant)
        if (isdigit((unsigned char)c)) d.push_back(c);
      while (d.size() > 1 && d.back() == '0') d.pop_back();
      *digits = d;
      *decpt = exp10 + 1;
      return;
    }
  }
}

std::string py_repr_double(double x) {
  if (std::isnan(x)) return "nan";
  if (std::isinf(x)) return x > 0 ? "inf" : "-inf";
  std::string sign = std::signbit(x) ? "-" : "";
  double ax = std::fabs(x);
  if (ax == 0.0) return sign + "0.0";
  std::string d;
  int decpt;
  shortest_digits(ax, &d, &decpt);
  std::string out;
  if (decpt <= -4 || decpt > 16) {  // repr switches to exponent form
    out = d.substr(0, 1);
    if (d.size() > 1) out += "." + d.substr(1);
    int e = decpt - 1;
    char buf[16];
    snprintf(buf, sizeof buf, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out += buf;
  } else if (decpt <= 0) {
    out = "0." + std::string((size_t)(-decpt), '0') + d;
  } else if ((size_t)decpt >= d.size()) {
    out = d + std::string((size_t)decpt - d.size(), '0') + ".0";
  } else {
    out = d.substr(0, (size_t)decpt) + "." + d.substr((size_t)decpt);
  }
  return sign + out;
}

// ---------------------------------------------------------------------------
// SHA-256 (FIPS 180-4), for the graph key digest (graph.py:133)
// ---------------------------------------------------------------------------
namespace {
const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
    0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
    0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
    0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
    0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
    0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
    0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};
inline uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
}  // namespace

std::string sha256_hex(const std::string& data) {
  uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  std::string msg = data;
  uint64_t bitlen = (uint64_t)data.size() * 8;
  msg.push_back((char)0x80);
  while (msg.size() % 64 != 56) msg.push_back((char)0);
  for (int i = 7; i >= 0; --i) msg.push_back((char)((bitlen >> (8 * i)) & 0xff));
  for (size_t blk = 0; blk < msg.size(); blk += 64) {
    uint32_t w[64];
    for (int i = 0; i < 16; ++i) {
      const unsigned char* p = (const unsigned char*)msg.data() + blk + 4 * i;
      w[i] = ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | p[3];
    }
    for (int i = 16; i < 64; ++i) {
      uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
      uint32_t ch = (e & f) ^ (~e & g);
      uint32_t t1 = hh + S1 + ch + K256[i] + w[i];
      uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
      uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
      uint32_t t2 = S0 + mj;
      hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
  }
  char out[65];
  for (int i = 0; i < 8; ++i) snprintf(out + 8 * i, 9, "%08x", h[i]);
  return std::string(out, 64);
}

// ---------------------------------------------------------------------------
// Topology
// ---------------------------------------------------------------------------

static std::string link_prefix(int a, int b) {
  return "link " + device_label(a) + "-" + device_label(b);
}

// LinkSpec.__post_init__ (topology.py:79-90); the message order matters.
static void validate_link(const mp_link& l) {
  const bool duplex_ok = l.duplex == MP_DUPLEX_FULL || l.duplex == MP_DUPLEX_HALF;
  if (l.bandwidth <= 0) throw err(MP_ERR_TOPOLOGY, link_prefix(l.a, l.b) + ": bandwidth must be > 0");
  if (l.latency < 0) throw err(MP_ERR_TOPOLOGY, link_prefix(l.a, l.b) + ": latency must be >= 0");
  if (!duplex_ok) throw err(MP_ERR_TOPOLOGY, link_prefix(l.a, l.b) + ": duplex must be full or half");
  if (l.sublinks < 1) throw err(MP_ERR_TOPOLOGY, link_prefix(l.a, l.b) + ": sublinks must be >= 1");
  if (l.a == l.b)
    throw err(MP_ERR_TOPOLOGY, "link endpoints must differ, got " + device_label(l.a) + "-" +
                                   device_label(l.b));
}

Topology Topology::build(const std::string& name, int n_accel, const std::vector<mp_link>& links) {
  Topology t;
  t.name = name;
  if (n_accel < 1) throw err(MP_ERR_TOPOLOGY, "topology needs at least one accelerator");
  t.n_accel = n_accel;
  t.links = links;
  std::set<std::pair<int, int>> seen;
  for (const mp_link& l : links) {
    for (int dev : {l.a, l.b})
      if (!(dev == MP_HOST || (dev >= 0 && dev < n_accel)))
        throw err(MP_ERR_TOPOLOGY, "link references unknown device " + device_label(dev));
    std::pair<int, int> pair(std::min(l.a, l.b), std::max(l.a, l.b));
    if (seen.count(pair))
      throw err(MP_ERR_TOPOLOGY,
                "duplicate link for pair " + device_label(l.a) + "-" + device_label(l.b));
    seen.insert(pair);
    std::string a = device_label(l.a), b = device_label(l.b);
    if (l.duplex == MP_DUPLEX_FULL) {
      auto fwd = std::make_pair(l.a, l.b), rev = std::make_pair(l.b, l.a);
      // dict assignment keeps the first insertion position of a key
      t.channels.push_back(Channel{a + "->" + b, l.bandwidth, l.latency, l.a, l.b});
      t.by_pair[fwd] = (int)t.channels.size() - 1;
      t.channels.push_back(Channel{b + "->" + a, l.bandwidth, l.latency, l.b, l.a});
      t.by_pair[rev] = (int)t.channels.size() - 1;
    } else {
      t.channels.push_back(Channel{a + "<->" + b, l.bandwidth, l.latency, l.a, l.b});
      t.by_pair[std::make_pair(l.a, l.b)] = (int)t.channels.size() - 1;
      t.by_pair[std::make_pair(l.b, l.a)] = (int)t.channels.size() - 1;
    }
  }
  return t;
}

int Topology::channel_for(int src, int dst) const {
  if (src == dst) throw err(MP_ERR_TOPOLOGY, "no self-link on device " + device_label(src));
  auto it = by_pair.find(std::make_pair(src, dst));
  if (it == by_pair.end())
    throw err(MP_ERR_TOPOLOGY, "no link joins " + device_label(src) + " and " +
                                   device_label(dst) + " in " + py_repr_str(name));
  return it->second;
}

Topology parse_topology(const std::string& source, const std::string& default_name) {
  enum { NONE, DEVICE, LINK, HOSTLINK } section = NONE;
  std::string name = default_name;
  std::vector<long long> accel;
  struct RawLink { long long a, b; double bw, lat; std::string duplex; long long subs; std::string where; };
  struct RawHost { long long dev; double bw, lat; std::string duplex; std::string where; };
  std::vector<RawLink> raw_links;
  std::vector<RawHost> raw_hosts;

  auto lines = py_splitlines(source);
  for (size_t ln = 0; ln < lines.size(); ++ln) {
    std::string raw = lines[ln];
    size_t hash = raw.find('#');
    std::string line = py_strip(hash == std::string::npos ? raw : raw.substr(0, hash));
    if (line.empty()) continue;
    std::string where = "line " + std::to_string(ln + 1);
    if (line.front() == '[' && line.back() == ']') {
      std::string sec = py_strip(line.substr(1, line.size() - 2));
      for (auto& c : sec) c = (char)tolower((unsigned char)c);
      if (sec == "device") section = DEVICE;
      else if (sec == "link") section = LINK;
      else if (sec == "hostlink") section = HOSTLINK;
      else throw err(MP_ERR_TOPOLOGY, where + ": unknown section [" + sec + "]");
      continue;
    }
    auto fields = py_split(line);
    auto expect = [&](size_t n) {
      if (fields.size() != n)
        throw err(MP_ERR_TOPOLOGY, where + ": expected " + std::to_string(n) + " fields, got " +
                                       std::to_string(fields.size()) + " in " + py_repr_str(line));
    };
    auto as_int = [&](const std::string& s) {
      long long v;
      if (!py_int(s, &v)) throw err(MP_ERR_TOPOLOGY, where + ": expected integer, got " + py_repr_str(s));
      return v;
    };
    auto as_float = [&](const std::string& s) {
      double v;
      if (!py_float(s, &v)) throw err(MP_ERR_TOPOLOGY, where + ": expected number, got " + py_repr_str(s));
      return v;
    };
    if (section == NONE) {
      if (fields[0] == "name" && fields.size() == 2) {
        name = fields[1];
        continue;
      }
      throw err(MP_ERR_TOPOLOGY, where + ": content before any section: " + py_repr_str(line));
    }
    if (section == DEVICE) {
      expect(2);
      if (fields[1] != "accelerator")
        throw err(MP_ERR_TOPOLOGY, where + ": only accelerator devices are declared; "
                                           "the host device is implicit");
      accel.push_back(as_int(fields[0]));
    } else if (section == LINK) {
      expect(6);
      RawLink r;
      r.a = as_int(fields[0]);
      r.b = as_int(fields[1]);
      r.bw = as_float(fields[2]);
      r.lat = as_float(fields[3]);
      r.duplex = fields[4];
      r.subs = as_int(fields[5]);
      r.where = where;
      raw_links.push_back(r);
    } else {
      expect(4);
      RawHost r;
      r.dev = as_int(fields[0]);
      r.bw = as_float(fields[1]);
      r.lat = as_float(fields[2]);
      r.duplex = fields[3];
      r.where = where;
      raw_hosts.push_back(r);
    }
  }
  std::vector<long long> sorted = accel;
  std::sort(sorted.begin(), sorted.end());
  for (size_t i = 0; i < sorted.size(); ++i) {
    if (sorted[i] != (long long)i) {
      std::string lst = "[";
      for (size_t k = 0; k < sorted.size(); ++k) lst += (k ? ", " : "") + std::to_string(sorted[k]);
      throw err(MP_ERR_TOPOLOGY, "accelerator indices must be dense 0..N-1, got " + lst + "]");
    }
  }
  if (accel.empty()) throw err(MP_ERR_TOPOLOGY, "no [device] entries found");
  long long n = (long long)accel.size();
  std::vector<mp_link> links;
  for (const RawLink& r : raw_links) {
    if (!(0 <= r.a && r.a < n && 0 <= r.b && r.b < n))
      throw err(MP_ERR_TOPOLOGY, r.where + ": link endpoint out of range: " + std::to_string(r.a) +
                                     "-" + std::to_string(r.b));
    mp_link l{};
    l.a = (int)r.a;
    l.b = (int)r.b;
    l.bandwidth = r.bw * (double)r.subs;  // topology.py:226 aggregate over sublinks
    l.latency = r.lat;
    l.duplex = r.duplex == "full" ? MP_DUPLEX_FULL : r.duplex == "half" ? MP_DUPLEX_HALF : -1;
    l.sublinks = (int)std::max<long long>(std::min<long long>(r.subs, 1LL << 30), -(1LL << 30));
    try {
      validate_link(l);
    } catch (const Error& e) {
      throw err(MP_ERR_TOPOLOGY, r.where + ": " + e.msg);
    }
    links.push_back(l);
  }
  std::set<long long> hostlinked;
  for (const RawHost& r : raw_hosts) {
    if (!(0 <= r.dev && r.dev < n))
      throw err(MP_ERR_TOPOLOGY, r.where + ": hostlink device out of range: " + std::to_string(r.dev));
    if (hostlinked.count(r.dev))
      throw err(MP_ERR_TOPOLOGY, r.where + ": duplicate hostlink for device " + std::to_string(r.dev));
    hostlinked.insert(r.dev);
    mp_link l{};
    l.a = (int)r.dev;
    l.b = MP_HOST;
    l.bandwidth = r.bw;
    l.latency = r.lat;
    l.duplex = r.duplex == "full" ? MP_DUPLEX_FULL : r.duplex == "half" ? MP_DUPLEX_HALF : -1;
    l.sublinks = 1;
    try {
      validate_link(l);
    } catch (const Error& e) {
      throw err(MP_ERR_TOPOLOGY, r.where + ": " + e.msg);
    }
    links.push_back(l);
  }
  return Topology::build(name, (int)n, links);
}

// ---------------------------------------------------------------------------
// Planner
// ---------------------------------------------------------------------------

// builtin sum() over floats on CPython >= 3.12: Neumaier compensated sum
// (bltinmodule.c builtin_sum_impl), started from int 0 so f = 0 + x0.
double py_sum(const std::vector<double>& xs) {
  if (xs.empty()) return 0.0;
  double f = 0.0 + xs[0];
  double c = 0.0;
  for (size_t i = 1; i < xs.size(); ++i) {
    double x = xs[i];
    double t = f + x;
    if (std::fabs(f) >= std::fabs(x)) c += (f - t) + x;
    else c += (x - t) + f;
    f = t;
  }
  if (c != 0.0 && std::isfinite(c)) f += c;
  return f;
}

void validate_config(const mp_config& cfg) {  // paths.py:78-86
  if (cfg.num_gpu_paths < 1) throw err(MP_ERR_PLAN, "num_gpu_paths must be >= 1");
  if (cfg.max_chunks < 1) throw err(MP_ERR_PLAN, "max_chunks must be >= 1");
  if (cfg.cache_capacity < 1) throw err(MP_ERR_PLAN, "cache_capacity must be >= 1");
  if (cfg.share_policy != MP_SHARE_BANDWIDTH && cfg.share_policy != MP_SHARE_EQUAL)
    throw err(MP_ERR_PLAN, "unknown share policy " + std::to_string(cfg.share_policy));
}

static double bottleneck(const Topology& t, const mp_path& p) {  // paths.py:62-64
  double m = t.channels[p.hops[0].channel].bandwidth;
  for (int h = 1; h < p.nhops; ++h) {
    double b = t.channels[p.hops[h].channel].bandwidth;
    if (b < m) m = b;  // builtin min keeps the first unless a later one is smaller
  }
  return m;
}

static mp_path make_path(int kind, int stage) {
  mp_path p{};
  p.kind = kind;
  p.stage = stage;
  p.share = 0.0;
  return p;
}

static void check_share(double s) {  // Path.__post_init__ paths.py:59-60
  if (!(0.0 <= s && s <= 1.0))
    throw err(MP_ERR_PLAN, "path share must lie in [0,1], got " + py_repr_double(s));
}

void validate_pathset(const mp_path* paths, int n) {  // paths.py:125-132
  std::vector<double> shares;
  for (int i = 0; i < n; ++i) shares.push_back(paths[i].share);
  double total = py_sum(shares);
  if (std::fabs(total - 1.0) > 1e-12)
    throw err(MP_ERR_PLAN, "path shares must sum to 1, got " + py_repr_double(total));
  std::set<int> stages;
  int count = 0, host = 0;
  for (int i = 0; i < n; ++i) {
    if (paths[i].stage != MP_NO_STAGE) {
      stages.insert(paths[i].stage);
      ++count;
    }
    if (paths[i].kind == MP_PATH_HOST) ++host;
  }
  if ((int)stages.size() != count) throw err(MP_ERR_PLAN, "staging devices must be pairwise distinct");
  if (host > 1) throw err(MP_ERR_PLAN, "at most one host-staged path per transfer");
}

// paths.py:153-167 _staged_path / _build_path_set, :144-150 _assign_shares
static std::vector<mp_path> build_path_set(const Topology& t, int src, int dst,
                                           const std::vector<int>& stages, const mp_config& cfg) {
  std::vector<mp_path> paths;
  mp_path d = make_path(MP_PATH_DIRECT, MP_NO_STAGE);
  d.nhops = 1;
  d.hops[0] = mp_hop{t.channel_for(src, dst), src, dst};
  paths.push_back(d);
  auto staged = [&](int stage, int kind) {
    mp_path p = make_path(kind, stage);
    p.nhops = 2;
    p.hops[0] = mp_hop{t.channel_for(src, stage), src, stage};
    p.hops[1] = mp_hop{t.channel_for(stage, dst), stage, dst};
    return p;
  };
  for (int s : stages) paths.push_back(staged(s, MP_PATH_GPU));
  if (cfg.host_path_enabled) paths.push_back(staged(MP_HOST, MP_PATH_HOST));
  std::vector<double> w;
  for (const mp_path& p : paths) w.push_back(cfg.share_policy == MP_SHARE_EQUAL ? 1.0 : bottleneck(t, p));
  double total = py_sum(w);
  for (size_t i = 0; i < paths.size(); ++i) {
    paths[i].share = w[i] / total;
    check_share(paths[i].share);
  }
  validate_pathset(paths.data(), (int)paths.size());
  return paths;
}

static bool is_accel(const Topology& t, int d) { return d >= 0 && d < t.n_accel; }

std::vector<mp_path> plan_paths(const Topology& t, int src, int dst, const mp_config& cfg) {
  validate_config(cfg);
  if (src == dst)
    throw err(MP_ERR_PLAN, "source and destination are the same device (" + device_label(src) + ")");
  if (src == MP_HOST || dst == MP_HOST) throw err(MP_ERR_PLAN, "transfers run between accelerators");
  std::vector<int> cand;
  for (int d = 0; d < t.n_accel; ++d)
    if (d != src && d != dst) cand.push_back(d);
  int needed = cfg.num_gpu_paths - 1;
  if (needed > (int)cand.size())
    throw err(MP_ERR_PLAN, std::to_string(cfg.num_gpu_paths) + " GPU paths need " +
                               std::to_string(needed) + " staging accelerators, only " +
                               std::to_string(cand.size()) + " available");
  (void)is_accel;
  return build_path_set(t, src, dst, std::vector<int>(cand.begin(), cand.begin() + needed), cfg);
}

// itertools.combinations(pool, r) in lexicographic index order
static std::vector<std::vector<int>> combinations(const std::vector<int>& pool, int r) {
  std::vector<std::vector<int>> out;
  int n = (int)pool.size();
  if (r > n) return out;
  std::vector<int> idx(r);
  for (int i = 0; i < r; ++i) idx[i] = i;
  while (true) {
    std::vector<int> c;
    for (int i : idx) c.push_back(pool[i]);
    out.push_back(c);
    int i = r - 1;
    while (i >= 0 && idx[i] == i + n - r) --i;
    if (i < 0) break;
    ++idx[i];
    for (int j = i + 1; j < r; ++j) idx[j] = idx[j - 1] + 1;
  }
  return out;
}

static std::vector<int> pathset_channels(const std::vector<mp_path>& ps) {  // paths.py:134-141
  std::vector<int> out;
  for (const mp_path& p : ps)
    for (int h = 0; h < p.nhops; ++h)
      if (std::find(out.begin(), out.end(), p.hops[h].channel) == out.end())
        out.push_back(p.hops[h].channel);
  return out;
}

// paths.py:210-242 plan_contention_free
std::vector<std::vector<mp_path>> plan_contention_free_sets(
    const Topology& t, const std::vector<std::pair<int, int>>& transfers, const mp_config& cfg,
    int* shared_out) {
  validate_config(cfg);
  if (transfers.empty()) throw err(MP_ERR_PLAN, "transfer list is empty");
  std::vector<std::vector<std::vector<int>>> options;
  for (auto& tr : transfers) {
    if (tr.first == tr.second)
      throw err(MP_ERR_PLAN,
                "source and destination are the same device (" + device_label(tr.first) + ")");
    std::vector<int> cand;
    for (int d = 0; d < t.n_accel; ++d)
      if (d != tr.first && d != tr.second) cand.push_back(d);
    int needed = cfg.num_gpu_paths - 1;
    if (needed > (int)cand.size())
      throw err(MP_ERR_PLAN, "transfer " + device_label(tr.first) + "->" + device_label(tr.second) +
                                 ": not enough staging accelerators");
    options.push_back(combinations(cand, needed));
  }
  size_t nt = transfers.size();
  std::vector<size_t> idx(nt, 0);
  std::vector<std::vector<mp_path>> best;
  int best_count = -1;
  std::vector<int> users(t.channels.size());
  while (true) {
    std::vector<std::vector<mp_path>> sets;
    for (size_t i = 0; i < nt; ++i)
      sets.push_back(build_path_set(t, transfers[i].first, transfers[i].second, options[i][idx[i]], cfg));
    std::fill(users.begin(), users.end(), 0);
    for (auto& ps : sets)
      for (int ch : pathset_channels(ps)) users[ch] += 1;
    int count = 0;
    for (int u : users) count += u > 1;
    if (best_count < 0 || count < best_count) {
      best = sets;
      best_count = count;
      if (count == 0) break;
    }
    // itertools.product: last position varies fastest
    int k = (int)nt - 1;
    while (k >= 0 && ++idx[k] == options[k].size()) idx[k--] = 0;
    if (k < 0) break;
  }
  *shared_out = best_count;
  return best;
}

// pipeline.py:51-78 make_chunk_plan
std::vector<mp_chunk> make_chunk_plan(const mp_path* paths, int n, int64_t size, int max_chunks) {
  if (size < 1)
    throw err(MP_ERR_CHUNK, "message size must be >= 1 byte, got " + std::to_string(size));
  if (max_chunks < 1)
    throw err(MP_ERR_CHUNK, "max_chunks must be >= 1, got " + std::to_string(max_chunks));
  std::vector<int> active;
  for (int p = 0; p < n; ++p)
    if (paths[p].share > 0.0) active.push_back(p);
  if (active.empty()) throw err(MP_ERR_CHUNK, "path set has no path with a positive share");
  std::vector<uint64_t> nominal(n, 0);
  for (int p : active) {
    // math.ceil(size * share / max_chunks): int*float and float/int in binary64
    double v = (double)size * paths[p].share / (double)max_chunks;
    nominal[p] = (uint64_t)std::ceil(v);
  }
  std::vector<mp_chunk> chunks;
  std::vector<int> seq(n, 0);
  uint64_t offset = 0, usize = (uint64_t)size;
  while (offset < usize) {
    for (int p : active) {
      if (offset >= usize) break;
      uint64_t length = std::min(nominal[p], usize - offset);
      if (length < 1) throw err(MP_ERR_CHUNK, "chunk length must be >= 1, got " + std::to_string(length));
      chunks.push_back(mp_chunk{offset, length, p, seq[p]});
      seq[p] += 1;
      offset += length;
    }
  }
  return chunks;
}

// pipeline.py:102-125 lane_schedule
LaneSchedule lane_schedule(const mp_path* paths, int n, const mp_chunk* chunks, int nc) {
  LaneSchedule s;
  std::vector<std::vector<int>> lane_of(n);
  int nl = 0;
  for (int p = 0; p < n; ++p)
    for (int h = 0; h < paths[p].nhops; ++h) lane_of[p].push_back(nl++);
  std::vector<std::vector<int32_t>> members(nl);
  for (int c = 0; c < nc; ++c) {
    int p = chunks[c].path_index;
    if (p < 0 || p >= n) throw err(MP_ERR_VALUE, "chunk path index out of range");
    if (paths[p].kind == MP_PATH_DIRECT) {
      members[lane_of[p][0]].push_back(c);
    } else {
      int l1 = lane_of[p][0], l2 = lane_of[p][1];
      members[l1].push_back(c);
      members[l2].push_back(c);
      int pos = (int)members[l1].size() - 1;
      s.deps.push_back(mp_lane_dep{l1, pos, l2, pos});
    }
  }
  for (int p = 0; p < n; ++p)
    for (int h = 0; h < paths[p].nhops; ++h) {
      int lid = lane_of[p][h];
      mp_lane lane{lid, p, h, (int32_t)s.members.size(), (int32_t)members[lid].size()};
      s.members.insert(s.members.end(), members[lid].begin(), members[lid].end());
      s.lanes.push_back(lane);
    }
  return s;
}

// graph.py:91-118 build_graph
LogicalGraph build_graph(const mp_path* paths, int n, const mp_chunk* chunks, int nc) {
  LaneSchedule s = lane_schedule(paths, n, chunks, nc);
  std::vector<std::vector<int>> lane_of(n);
  for (const mp_lane& l : s.lanes) {
    if ((int)lane_of[l.path_index].size() <= l.hop) lane_of[l.path_index].resize(l.hop + 1);
    lane_of[l.path_index][l.hop] = l.lane_id;
  }
  LogicalGraph g;
  g.lane_count = (int)s.lanes.size();
  for (int c = 0; c < nc; ++c) {
    const mp_chunk& ch = chunks[c];
    const mp_path& p = paths[ch.path_index];
    if (p.kind == MP_PATH_DIRECT) {
      const mp_hop& h = p.hops[0];
      g.nodes.push_back(mp_node{(int32_t)g.nodes.size(), h.src, h.dst, h.channel, ch.offset,
                                ch.length, lane_of[ch.path_index][0], MP_ROLE_DIRECT, c,
                                ch.path_index});
    } else {
      const mp_hop& h1 = p.hops[0];
      const mp_hop& h2 = p.hops[1];
      int first = (int)g.nodes.size();
      g.nodes.push_back(mp_node{first, h1.src, h1.dst, h1.channel, ch.offset, ch.length,
                                lane_of[ch.path_index][0], MP_ROLE_HOP1, c, ch.path_index});
      g.nodes.push_back(mp_node{first + 1, h2.src, h2.dst, h2.channel, ch.offset, ch.length,
                                lane_of[ch.path_index][1], MP_ROLE_HOP2, c, ch.path_index});
      g.edges.push_back(mp_edge{first, first + 1});
    }
  }
  return g;
}

// graph.py:132-144: sha256(repr((cfg fields, src, dst, paths)).encode())
std::string graph_digest(const std::vector<std::string>& channel_ids, const mp_config& cfg,
                         int src, int dst, const mp_path* paths, int n) {
  static const char* kinds[] = {"direct", "gpu", "host"};
  std::string r = "(";
  r += std::to_string(cfg.num_gpu_paths) + ", ";
  r += std::string(cfg.host_path_enabled ? "True" : "False") + ", ";
  r += std::to_string(cfg.max_chunks) + ", ";
  r += std::string(cfg.graph_mode ? "True" : "False") + ", ";
  r += py_repr_str(cfg.share_policy == MP_SHARE_EQUAL ? "equal" : "bandwidth_proportional") + ", ";
  r += py_repr_str(device_label(src)) + ", " + py_repr_str(device_label(dst)) + ", (";
  for (int i = 0; i < n; ++i) {
    const mp_path& p = paths[i];
    r += "(" + py_repr_str(kinds[p.kind]) + ", ";
    r += (p.stage == MP_NO_STAGE ? std::string("None") : py_repr_str(device_label(p.stage))) + ", ";
    r += py_repr_double(p.share) + ", (";
    for (int h = 0; h < p.nhops; ++h) {
      r += py_repr_str(channel_ids[p.hops[h].channel]);
      if (p.nhops == 1 || h + 1 < p.nhops) r += p.nhops == 1 ? "," : ", ";
    }
    r += "))";
    if (n == 1 || i + 1 < n) r += n == 1 ? "," : ", ";
  }
  r += "))";
  return sha256_hex(r);
}

}  // namespace mp

// ===========================================================================
// C ABI
// ===========================================================================
using namespace mp;

// LRU keyed by byte strings (graph.py:147-186: OrderedDict, move_to_end on a
// hit, popitem(last=False) while over capacity).
struct mp_cache {
  int capacity;
  std::list<std::pair<std::string, uint64_t>> order;  // LRU first
  std::unordered_map<std::string, std::list<std::pair<std::string, uint64_t>>::iterator> index;
};

template <typename T>
static int copy_out(const std::vector<T>& v, T* out, int32_t cap, int32_t* n_out) {
  if (n_out) *n_out = (int32_t)v.size();
  if ((int32_t)v.size() > cap || (!out && !v.empty()))
    return fail(MP_ERR_CAPACITY, "output capacity " + std::to_string(cap) + " < " +
                                     std::to_string(v.size()));
  if (!v.empty()) memcpy(out, v.data(), v.size() * sizeof(T));
  return MP_OK;
}

#define MP_GUARD_BEGIN try {
#define MP_GUARD_END                                       \
  }                                                        \
  catch (const Error& e) {                                 \
    return fail(e.code, e.msg);                            \
  }                                                        \
  catch (const std::exception& e) {                        \
    return fail(MP_ERR_VALUE, e.what());                   \
  }

extern "C" {

const char* mp_last_error(void) { return g_last_error.c_str(); }
int mp_abi_version(void) { return MP_ABI_VERSION; }

int mp_topology_load(const char* text, const char* default_name, mp_topology** out) {
  MP_GUARD_BEGIN
  if (!text || !out) return fail(MP_ERR_VALUE, "null argument");
  auto* t = new mp_topology{parse_topology(text, default_name ? default_name : "topology")};
  *out = t;
  return MP_OK;
  MP_GUARD_END
}

int mp_topology_create(const char* name, int32_t n_accel, const mp_link* links, int32_t n_links,
                       mp_topology** out) {
  MP_GUARD_BEGIN
  if (!out || (n_links > 0 && !links)) return fail(MP_ERR_VALUE, "null argument");
  std::vector<mp_link> v(links, links + n_links);
  *out = new mp_topology{Topology::build(name ? name : "topology", n_accel, v)};
  return MP_OK;
  MP_GUARD_END
}

void mp_topology_destroy(mp_topology* topo) { delete topo; }

int mp_topology_info(const mp_topology* topo, int32_t* n_accel, int32_t* n_links,
                     int32_t* n_channels) {
  if (!topo) return fail(MP_ERR_VALUE, "null topology");
  if (n_accel) *n_accel = topo->t.n_accel;
  if (n_links) *n_links = (int32_t)topo->t.links.size();
  if (n_channels) *n_channels = (int32_t)topo->t.channels.size();
  return MP_OK;
}

int mp_topology_name(const mp_topology* topo, char* buf, size_t cap) {
  if (!topo || !buf || cap == 0) return fail(MP_ERR_VALUE, "null argument");
  if (topo->t.name.size() + 1 > cap) return fail(MP_ERR_CAPACITY, "name buffer too small");
  memcpy(buf, topo->t.name.c_str(), topo->t.name.size() + 1);
  return MP_OK;
}

int mp_topology_link(const mp_topology* topo, int32_t i, mp_link* out) {
  if (!topo || !out) return fail(MP_ERR_VALUE, "null argument");
  if (i < 0 || i >= (int)topo->t.links.size()) return fail(MP_ERR_VALUE, "link index out of range");
  *out = topo->t.links[i];
  return MP_OK;
}

int mp_topology_channel(const mp_topology* topo, int32_t i, mp_channel* out) {
  if (!topo || !out) return fail(MP_ERR_VALUE, "null argument");
  if (i < 0 || i >= (int)topo->t.channels.size()) return fail(MP_ERR_VALUE, "channel index out of range");
  const Channel& c = topo->t.channels[i];
  memset(out, 0, sizeof *out);
  snprintf(out->id, sizeof out->id, "%s", c.id.c_str());
  out->bandwidth = c.bandwidth;
  out->latency = c.latency;
  out->a = c.a;
  out->b = c.b;
  return MP_OK;
}

int mp_topology_channel_for(const mp_topology* topo, int32_t src, int32_t dst, int32_t* channel) {
  MP_GUARD_BEGIN
  if (!topo || !channel) return fail(MP_ERR_VALUE, "null argument");
  *channel = topo->t.channel_for(src, dst);
  return MP_OK;
  MP_GUARD_END
}

int mp_config_validate(const mp_config* cfg) {
  MP_GUARD_BEGIN
  if (!cfg) return fail(MP_ERR_VALUE, "null config");
  validate_config(*cfg);
  return MP_OK;
  MP_GUARD_END
}

int mp_plan_paths(const mp_topology* topo, int32_t src, int32_t dst, const mp_config* cfg,
                  mp_path* out, int32_t cap, int32_t* n_out) {
  MP_GUARD_BEGIN
  if (!topo || !cfg) return fail(MP_ERR_VALUE, "null argument");
  return copy_out(plan_paths(topo->t, src, dst, *cfg), out, cap, n_out);
  MP_GUARD_END
}

int mp_plan_contention_free(const mp_topology* topo, const int32_t* srcs, const int32_t* dsts,
                            int32_t n_transfers, const mp_config* cfg, mp_path* out, int32_t cap,
                            int32_t* paths_per_set, int32_t* shared) {
  MP_GUARD_BEGIN
  if (!topo || !cfg || (n_transfers > 0 && (!srcs || !dsts))) return fail(MP_ERR_VALUE, "null argument");
  std::vector<std::pair<int, int>> tr;
  for (int i = 0; i < n_transfers; ++i) tr.emplace_back(srcs[i], dsts[i]);
  int sh = 0;
  auto sets = plan_contention_free_sets(topo->t, tr, *cfg, &sh);
  std::vector<mp_path> flat;
  for (auto& s : sets) flat.insert(flat.end(), s.begin(), s.end());
  if (paths_per_set) *paths_per_set = sets.empty() ? 0 : (int32_t)sets[0].size();
  if (shared) *shared = sh;
  int32_t n = 0;
  return copy_out(flat, out, cap, &n);
  MP_GUARD_END
}

int mp_pathset_validate(const mp_path* paths, int32_t n) {
  MP_GUARD_BEGIN
  if (n > 0 && !paths) return fail(MP_ERR_VALUE, "null argument");
  validate_pathset(paths, n);
  return MP_OK;
  MP_GUARD_END
}

int mp_make_chunk_plan(const mp_path* paths, int32_t n_paths, uint64_t size, int32_t max_chunks,
                       mp_chunk* out, int32_t cap, int32_t* n_out) {
  MP_GUARD_BEGIN
  if (n_paths > 0 && !paths) return fail(MP_ERR_VALUE, "null argument");
  return copy_out(make_chunk_plan(paths, n_paths, (int64_t)size, max_chunks), out, cap, n_out);
  MP_GUARD_END
}

int mp_lane_schedule(const mp_path* paths, int32_t n_paths, const mp_chunk* chunks,
                     int32_t n_chunks, mp_lane* lanes, int32_t lanes_cap, int32_t* n_lanes,
                     int32_t* members, int32_t members_cap, int32_t* n_members,
                     mp_lane_dep* deps, int32_t deps_cap, int32_t* n_deps) {
  MP_GUARD_BEGIN
  LaneSchedule s = lane_schedule(paths, n_paths, chunks, n_chunks);
  int rc = copy_out(s.lanes, lanes, lanes_cap, n_lanes);
  int rc2 = copy_out(s.members, members, members_cap, n_members);
  int rc3 = copy_out(s.deps, deps, deps_cap, n_deps);
  if (rc || rc2 || rc3) return fail(MP_ERR_CAPACITY, "lane schedule output capacity too small");
  return MP_OK;
  MP_GUARD_END
}

int mp_build_graph(const mp_path* paths, int32_t n_paths, const mp_chunk* chunks, int32_t n_chunks,
                   mp_node* nodes, int32_t nodes_cap, int32_t* n_nodes, mp_edge* edges,
                   int32_t edges_cap, int32_t* n_edges, int32_t* lane_count) {
  MP_GUARD_BEGIN
  LogicalGraph g = build_graph(paths, n_paths, chunks, n_chunks);
  if (lane_count) *lane_count = g.lane_count;
  int rc = copy_out(g.nodes, nodes, nodes_cap, n_nodes);
  int rc2 = copy_out(g.edges, edges, edges_cap, n_edges);
  if (rc || rc2) return fail(MP_ERR_CAPACITY, "graph output capacity too small");
  return MP_OK;
  MP_GUARD_END
}

int mp_graph_digest(const mp_config* cfg, int32_t src, int32_t dst, const mp_path* paths,
                    int32_t n_paths, const char* const* channel_ids, int32_t n_channels,
                    char* out_hex) {
  MP_GUARD_BEGIN
  if (!cfg || !out_hex || (n_paths > 0 && !paths) || (n_channels > 0 && !channel_ids))
    return fail(MP_ERR_VALUE, "null argument");
  std::vector<std::string> ids;
  for (int i = 0; i < n_channels; ++i) ids.push_back(channel_ids[i] ? channel_ids[i] : "");
  for (int i = 0; i < n_paths; ++i) {
    if (paths[i].kind < MP_PATH_DIRECT || paths[i].kind > MP_PATH_HOST || paths[i].nhops < 1 ||
        paths[i].nhops > 2)
      return fail(MP_ERR_VALUE, "malformed path");
    for (int h = 0; h < paths[i].nhops; ++h)
      if (paths[i].hops[h].channel < 0 || paths[i].hops[h].channel >= n_channels)
        return fail(MP_ERR_VALUE, "hop channel out of range");
  }
  std::string hex = graph_digest(ids, *cfg, src, dst, paths, n_paths);
  memcpy(out_hex, hex.c_str(), 65);
  return MP_OK;
  MP_GUARD_END
}

int mp_link_validate(const mp_link* link) {
  MP_GUARD_BEGIN
  if (!link) return fail(MP_ERR_VALUE, "null argument");
  validate_link(*link);
  return MP_OK;
  MP_GUARD_END
}

int mp_format_double(double x, char* buf, size_t cap) {
  std::string s = py_repr_double(x);
  if (!buf || s.size() + 1 > cap) return fail(MP_ERR_CAPACITY, "buffer too small");
  memcpy(buf, s.c_str(), s.size() + 1);
  return MP_OK;
}

int mp_cache_create(int32_t capacity, mp_cache** out) {
  if (!out) return fail(MP_ERR_VALUE, "null argument");
  if (capacity < 1)
    return fail(MP_ERR_VALUE, "cache capacity must be >= 1, got " + std::to_string(capacity));
  *out = new mp_cache{capacity, {}, {}};
  return MP_OK;
}

void mp_cache_destroy(mp_cache* cache) { delete cache; }

int mp_cache_access(mp_cache* cache, const void* key, size_t key_len, int32_t* hit,
                    uint64_t* value, uint64_t* evicted, int32_t evicted_cap, int32_t* n_evicted) {
  if (!cache || !hit || !value || (key_len && !key)) return fail(MP_ERR_VALUE, "null argument");
  std::string k((const char*)key, key_len);
  if (n_evicted) *n_evicted = 0;
  auto it = cache->index.find(k);
  if (it != cache->index.end()) {
    cache->order.splice(cache->order.end(), cache->order, it->second);  // move_to_end
    *hit = 1;
    *value = it->second->second;
    return MP_OK;
  }
  *hit = 0;
  cache->order.emplace_back(k, *value);
  cache->index[k] = std::prev(cache->order.end());
  int ne = 0;
  while ((int)cache->order.size() > cache->capacity) {  // popitem(last=False)
    if (evicted && ne < evicted_cap) evicted[ne] = cache->order.front().second;
    ++ne;
    cache->index.erase(cache->order.front().first);
    cache->order.pop_front();
  }
  if (n_evicted) *n_evicted = ne;
  return MP_OK;
}

int mp_cache_len(const mp_cache* cache, int32_t* n) {
  if (!cache || !n) return fail(MP_ERR_VALUE, "null argument");
  *n = (int32_t)cache->order.size();
  return MP_OK;
}

int mp_cache_contains(const mp_cache* cache, const void* key, size_t key_len, int32_t* yes) {
  if (!cache || !yes) return fail(MP_ERR_VALUE, "null argument");
  *yes = cache->index.count(std::string((const char*)key, key_len)) ? 1 : 0;
  return MP_OK;
}

int mp_cache_values(const mp_cache* cache, uint64_t* out, int32_t cap, int32_t* n_out) {
  if (!cache) return fail(MP_ERR_VALUE, "null argument");
  std::vector<uint64_t> v;
  for (auto& kv : cache->order) v.push_back(kv.second);
  return copy_out(v, out, cap, n_out);
}

}  // extern "C"
