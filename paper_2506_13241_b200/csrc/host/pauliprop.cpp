// pauliprop.cpp -- host side of the B200 engine: Pauli-string algebra and
// I/O, angles and circuits, geometries and the kicked-Ising builder, and the
// Engine / run_circuit front end over the C-ABI (include/pauliprop_gpu.h).
//
// Behaviour follows the reference API it stands in for; each block cites the
// reference function whose contract it keeps.
#include "pauliprop.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <iterator>
#include <sys/stat.h>
#include <fstream>
#include <limits>
#include <set>
#include <sstream>

#include "../../../include/pauliprop_gpu.h"

namespace pauliprop {

namespace {
constexpr double kPi = 3.14159265358979323846;

// su(2) structure constants on one site, rows a, columns b, codes I X Y Z
// (pauli_string.cpp:25-34): sigma_a sigma_b = i^{phase} sigma_{a xor b}.
constexpr int8_t kPhase[4][4] = {{0, 0, 0, 0}, {0, 0, 1, -1}, {0, -1, 0, 1}, {0, 1, -1, 0}};

uint64_t splitmix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void require_site(int site, int n) {
  if (site < 0 || site >= n)
    throw std::invalid_argument("pauli site index " + std::to_string(site) + " out of range for n=" +
                                std::to_string(n));
}

int code_of(char c) {
  switch (c) {
    case 'I': return 0;
    case 'X': return 1;
    case 'Y': return 2;
    case 'Z': return 3;
    default: return -1;
  }
}

std::string trim(const std::string& s) {
  size_t a = s.find_first_not_of(" \t\r");
  if (a == std::string::npos) return "";
  size_t b = s.find_last_not_of(" \t\r");
  return s.substr(a, b - a + 1);
}
}  // namespace

// ------------------------------------------------------------ algebra
PauliString single_site(int site, Pauli pauli) {
  require_site(site, kMaxQubits);
  PauliString s;
  s.set_code(site, static_cast<uint8_t>(pauli));
  return s;
}

uint64_t hash_string(const PauliString& s) {
  uint64_t h = 0;
  for (uint64_t w : s.words) h = splitmix(h ^ w);
  return h;
}

int local_phase(uint8_t a, uint8_t b) { return kPhase[a & 3][b & 3]; }

int phase_exponent(const PauliString& I, const PauliString& J, int n) {
  int b = 0;
  for (int site = 0; site < n; ++site) b += local_phase(I.code_at(site), J.code_at(site));
  return ((b % 4) + 4) % 4;
}

bool commutes(const PauliString& I, const PauliString& J, int n) { return (phase_exponent(I, J, n) & 1) == 0; }

StringProduct string_product(const PauliString& I, const PauliString& J, int n) {
  return {I ^ J, phase_exponent(I, J, n)};
}

int pauli_weight(const PauliString& s) {
  int w = 0;
  for (uint64_t v : s.words) w += __builtin_popcountll((v | (v >> 1)) & 0x5555555555555555ULL);
  return w;
}

// Dense ("IZIZ", leftmost = site n-1) or sparse ("Z2 Z0") labels,
// pauli_string.cpp:105-177.
PauliString parse_pauli_label(const std::string& text, int n) {
  if (n < 1 || n > kMaxQubits) throw std::invalid_argument("qubit count out of range: " + std::to_string(n));
  std::string t = trim(text);
  if (t.empty()) throw std::invalid_argument("empty pauli label");
  bool digit = t.find_first_of("0123456789") != std::string::npos;
  bool space = t.find_first_of(" \t") != std::string::npos;
  PauliString s;
  if (!digit && !space) {
    if ((int)t.size() != n)
      throw std::invalid_argument("dense pauli label \"" + t + "\" has length " + std::to_string(t.size()) +
                                  ", expected n=" + std::to_string(n));
    for (int i = 0; i < n; ++i) {
      int c = code_of(t[i]);
      if (c < 0) throw std::invalid_argument(std::string("invalid pauli character '") + t[i] + "'");
      s.set_code(n - 1 - i, (uint8_t)c);
    }
    return s;
  }
  std::istringstream in(t);
  std::string tok;
  while (in >> tok) {
    int c = code_of(tok[0]);
    if (c <= 0) throw std::invalid_argument("invalid sparse pauli token \"" + tok + "\"");
    if (tok.size() < 2) throw std::invalid_argument("sparse pauli token \"" + tok + "\" is missing a site index");
    size_t pos = 0;
    int site;
    try {
      site = std::stoi(tok.substr(1), &pos);
    } catch (const std::exception&) {
      throw std::invalid_argument("invalid site index in token \"" + tok + "\"");
    }
    if (pos + 1 != tok.size()) throw std::invalid_argument("invalid sparse pauli token \"" + tok + "\"");
    require_site(site, n);
    if (s.code_at(site)) throw std::invalid_argument("site " + std::to_string(site) + " appears twice in pauli label");
    s.set_code(site, (uint8_t)c);
  }
  return s;
}

std::string to_dense_label(const PauliString& s, int n) {
  std::string out(n, 'I');
  for (int site = 0; site < n; ++site) out[n - 1 - site] = "IXYZ"[s.code_at(site)];
  return out;
}

std::string to_sparse_label(const PauliString& s, int n) {
  std::string out;
  for (int site = 0; site < n; ++site) {
    uint8_t c = s.code_at(site);
    if (!c) continue;
    if (!out.empty()) out += ' ';
    out += "IXYZ"[c];
    out += std::to_string(site);
  }
  return out.empty() ? "I" : out;
}

std::string to_hex(const PauliString& s, int n) {
  int digits = (2 * n + 3) / 4;
  std::string out(digits, '0');
  for (int d = 0; d < digits; ++d) {
    int bit = 4 * d;
    out[digits - 1 - d] = "0123456789abcdef"[(s.words[bit >> 6] >> (bit & 63)) & 0xf];
  }
  return out;
}

PauliString from_hex(const std::string& hex, int n) {
  PauliString s;
  int bit = 0;
  for (auto it = hex.rbegin(); it != hex.rend(); ++it, bit += 4) {
    char c = (char)std::tolower(*it);
    int v;
    if (c >= '0' && c <= '9') v = c - '0';
    else if (c >= 'a' && c <= 'f') v = 10 + (c - 'a');
    else throw std::invalid_argument(std::string("invalid hex digit '") + *it + "'");
    if (v == 0) continue;
    if (bit >= 2 * kMaxQubits) throw std::invalid_argument("hex index wider than the maximum width");
    s.words[bit >> 6] |= (uint64_t)v << (bit & 63);
  }
  for (int site = n; site < kMaxQubits; ++site)
    if (s.code_at(site)) throw std::invalid_argument("hex index has bits above site " + std::to_string(n - 1));
  return s;
}

// ------------------------------------------------------------ angles
// Exact trig at half-integer multiples of pi (circuit.cpp:28-40).
static double cos_pi(double r) {
  double f = std::fmod(r, 2.0);
  if (f < 0) f += 2.0;
  double twice = 2.0 * f;
  if (twice == std::floor(twice)) {
    static constexpr double table[4] = {1.0, 0.0, -1.0, 0.0};
    return table[static_cast<int>(twice) & 3];
  }
  return std::cos(r * kPi);
}

Angle Angle::from_radians(double r) {
  Angle a;
  a.radians = r;
  return a;
}
Angle Angle::from_pi_units(double r) {
  Angle a;
  a.radians = r * kPi;
  a.in_pi_units = true;
  a.pi_units = r;
  return a;
}
double Angle::cosine() const { return in_pi_units ? cos_pi(pi_units) : std::cos(radians); }
double Angle::sine() const { return in_pi_units ? cos_pi(pi_units - 0.5) : std::sin(radians); }

Angle parse_angle(const std::string& text) {
  std::string t = text;
  bool pi = false;
  if (t.size() >= 2 && (t.ends_with("pi") || t.ends_with("PI"))) {
    pi = true;
    t = t.substr(0, t.size() - 2);
    if (t.empty() || t == "-" || t == "+") t += "1";
  }
  size_t pos = 0;
  double v;
  try {
    v = std::stod(t, &pos);
  } catch (const std::exception&) {
    throw std::invalid_argument("invalid angle \"" + text + "\"");
  }
  if (pos != t.size()) throw std::invalid_argument("invalid angle \"" + text + "\"");
  if (!std::isfinite(v)) throw std::invalid_argument("angle must be finite: \"" + text + "\"");
  return pi ? Angle::from_pi_units(v) : Angle::from_radians(v);
}

Gate::Gate(const PauliString& g, Angle a)
    : generator(g), theta(a.radians), cos_theta(a.cosine()), sin_theta(a.sine()) {}

size_t Circuit::total_gates() const {
  size_t t = 0;
  for (const auto& l : layers) t += l.size();
  return t;
}

// "label angle" per line, blank line = layer break, '#' comments
// (circuit.cpp:101-137).
Circuit parse_circuit_text(const std::string& text, int n) {
  Circuit c;
  c.n = n;
  std::vector<Gate> layer;
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    size_t h = line.find('#');
    if (h != std::string::npos) line = line.substr(0, h);
    size_t last = line.find_last_not_of(" \t\r");
    if (last == std::string::npos) {
      if (!layer.empty()) {
        c.layers.push_back(std::move(layer));
        layer.clear();
      }
      continue;
    }
    line = line.substr(0, last + 1);
    size_t split = line.find_last_of(" \t");
    if (split == std::string::npos)
      throw std::invalid_argument("circuit line " + std::to_string(lineno) + ": expected \"pauli-label angle\"");
    try {
      layer.emplace_back(parse_pauli_label(line.substr(0, split), n), parse_angle(line.substr(split + 1)));
    } catch (const std::invalid_argument& e) {
      throw std::invalid_argument("circuit line " + std::to_string(lineno) + ": " + e.what());
    }
  }
  if (!layer.empty()) c.layers.push_back(std::move(layer));
  return c;
}

std::string format_circuit(const Circuit& c) {
  std::ostringstream out;
  char buf[32];
  for (size_t l = 0; l < c.layers.size(); ++l) {
    if (l) out << '\n';
    for (const Gate& g : c.layers[l]) {
      std::snprintf(buf, sizeof(buf), "%.17g", g.theta);
      out << to_sparse_label(g.generator, c.n) << ' ' << buf << '\n';
    }
  }
  return out.str();
}

// ------------------------------------------------------------ geometry
// "i j [color]" lines (models.cpp:27-105): same validation rules.
Geometry load_geometry_text(const std::string& text) {
  Geometry g;
  std::set<std::pair<int, int>> seen;
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  bool any_color = false, any_plain = false;
  while (std::getline(in, line)) {
    ++lineno;
    size_t h = line.find('#');
    if (h != std::string::npos) line = line.substr(0, h);
    std::istringstream ls(line);
    int i, j;
    if (!(ls >> i)) continue;
    if (!(ls >> j)) throw std::invalid_argument("geometry line " + std::to_string(lineno) + ": expected \"i j [color]\"");
    int color = -1;
    if (ls >> color) {
      if (color < 0) throw std::invalid_argument("geometry line " + std::to_string(lineno) + ": negative color");
      any_color = true;
    } else {
      any_plain = true;
    }
    std::string trailing;
    ls.clear();
    if (ls >> trailing)
      throw std::invalid_argument("geometry line " + std::to_string(lineno) + ": trailing content \"" + trailing + "\"");
    if (i < 0 || j < 0) throw std::invalid_argument("geometry line " + std::to_string(lineno) + ": negative qubit index");
    if (i == j) throw std::invalid_argument("geometry line " + std::to_string(lineno) + ": self loop on qubit " + std::to_string(i));
    if (!seen.insert(std::minmax(i, j)).second)
      throw std::invalid_argument("geometry line " + std::to_string(lineno) + ": duplicate edge " + std::to_string(i) +
                                  "-" + std::to_string(j));
    g.edges.emplace_back(i, j);
    g.edge_colors.push_back(color);
    g.n = std::max({g.n, i + 1, j + 1});
  }
  if (g.edges.empty()) throw std::invalid_argument("geometry file has no edges");
  if (any_color && any_plain) throw std::invalid_argument("geometry file mixes colored and uncolored edges");
  if (!any_color) {
    g.edge_colors.clear();
    return g;
  }
  g.color_count = 1 + *std::max_element(g.edge_colors.begin(), g.edge_colors.end());
  std::vector<std::set<int>> used(g.color_count);
  for (size_t e = 0; e < g.edges.size(); ++e) {
    auto [i, j] = g.edges[e];
    auto& q = used[g.edge_colors[e]];
    if (!q.insert(i).second || !q.insert(j).second)
      throw std::invalid_argument("edges overlap within color " + std::to_string(g.edge_colors[e]) + " at edge " +
                                  std::to_string(i) + "-" + std::to_string(j));
  }
  return g;
}

Geometry load_geometry_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::invalid_argument("cannot open geometry file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return load_geometry_text(ss.str());
}

// Heavy-hex, 127 qubits, following the construction of BASELINE.json
// config 1: rows are numbered row-major with each gap's 4 bridge qubits
// interleaved after the row above it; row 0 has cols 0-13, rows 1-5 cols
// 0-14, row 6 cols 1-14; bridges sit at cols {0,4,8,12} below even rows and
// {2,6,10,14} below odd rows.  Edges are coloured by a deterministic
// backtracking 3-edge-colouring (no two edges of a colour share a qubit).
Geometry heavy_hex_127() {
  std::vector<std::vector<int>> row_q(7, std::vector<int>(15, -1));
  std::vector<std::array<int, 4>> bridge_q(6);
  int q = 0;
  for (int r = 0; r < 7; ++r) {
    int c0 = r == 6 ? 1 : 0, c1 = r == 0 ? 13 : 14;
    for (int c = c0; c <= c1; ++c) row_q[r][c] = q++;
    if (r < 6)
      for (int b = 0; b < 4; ++b) bridge_q[r][b] = q++;
  }
  std::vector<std::pair<int, int>> edges;
  for (int r = 0; r < 7; ++r)
    for (int c = 0; c < 14; ++c)
      if (row_q[r][c] >= 0 && row_q[r][c + 1] >= 0) edges.emplace_back(row_q[r][c], row_q[r][c + 1]);
  for (int r = 0; r < 6; ++r)
    for (int b = 0; b < 4; ++b) {
      int col = (r % 2 == 0 ? 0 : 2) + 4 * b;
      edges.emplace_back(row_q[r][col], bridge_q[r][b]);
      edges.emplace_back(bridge_q[r][b], row_q[r + 1][col]);
    }
  // 3-edge-colouring of this bipartite (all cycles have length 12), degree-3
  // graph by alternating-path recolouring (Koenig): colour edges in order;
  // if no colour is free at both ends, swap the (a, b) path from v.
  const int E = (int)edges.size();
  std::vector<int> color(E, -1);
  std::vector<std::array<int, 3>> at(q, {-1, -1, -1});  // at[v][c] = edge of colour c at v
  for (int e = 0; e < E; ++e) {
    auto [u, v] = edges[e];
    int a = -1, b = -1;
    for (int c = 0; c < 3 && a < 0; ++c)
      if (at[u][c] < 0) a = c;
    for (int c = 0; c < 3 && b < 0; ++c)
      if (at[v][c] < 0) b = c;
    if (at[v][a] >= 0) {
      // walk the path from v alternating colours a, b and swap them
      std::vector<int> path;
      int x = v, col = a;
      while (at[x][col] >= 0) {
        int pe = at[x][col];
        path.push_back(pe);
        x = edges[pe].first == x ? edges[pe].second : edges[pe].first;
        col = col == a ? b : a;
      }
      for (int pe : path) {
        at[edges[pe].first][color[pe]] = -1;
        at[edges[pe].second][color[pe]] = -1;
      }
      for (int pe : path) {
        color[pe] = color[pe] == a ? b : a;
        at[edges[pe].first][color[pe]] = pe;
        at[edges[pe].second][color[pe]] = pe;
      }
    }
    if (at[u][a] >= 0 || at[v][a] >= 0) throw std::logic_error("heavy-hex colouring failed");
    color[e] = a;
    at[u][a] = at[v][a] = e;
  }
  std::ostringstream text;
  for (int e = 0; e < E; ++e) text << edges[e].first << ' ' << edges[e].second << ' ' << color[e] << '\n';
  return load_geometry_text(text.str());
}

std::vector<int> bfs_ball(const Geometry& geom, int start, int radius) {
  std::vector<std::vector<int>> adj(geom.n);
  for (auto [i, j] : geom.edges) {
    adj[i].push_back(j);
    adj[j].push_back(i);
  }
  std::vector<int> dist(geom.n, -1);
  std::deque<int> qu{start};
  dist[start] = 0;
  while (!qu.empty()) {
    int u = qu.front();
    qu.pop_front();
    if (dist[u] == radius) continue;
    for (int v : adj[u])
      if (dist[v] < 0) {
        dist[v] = dist[u] + 1;
        qu.push_back(v);
      }
  }
  std::vector<int> ball;
  for (int i = 0; i < geom.n; ++i)
    if (dist[i] >= 0) ball.push_back(i);
  return ball;
}

// One Trotter step: X rotations on qubits 0..n-1 ascending, then ZZ
// rotations colour by colour in edge-list order (models.cpp:149-171).
std::vector<Gate> kicked_ising_layer(const Geometry& geom, Angle theta_x, Angle theta_zz) {
  std::vector<Gate> layer;
  layer.reserve(geom.n + geom.edges.size());
  for (int q = 0; q < geom.n; ++q) layer.emplace_back(single_site(q, Pauli::X), theta_x);
  auto add = [&](size_t e) {
    auto [i, j] = geom.edges[e];
    layer.emplace_back(single_site(i, Pauli::Z) ^ single_site(j, Pauli::Z), theta_zz);
  };
  if (geom.has_coloring()) {
    for (int c = 0; c < geom.color_count; ++c)
      for (size_t e = 0; e < geom.edges.size(); ++e)
        if (geom.edge_colors[e] == c) add(e);
  } else {
    for (size_t e = 0; e < geom.edges.size(); ++e) add(e);
  }
  return layer;
}

Circuit build_kicked_ising(const Geometry& geom, Angle theta_x, Angle theta_zz, int layers) {
  if (layers < 1) throw std::invalid_argument("layer count must be >= 1");
  Circuit c;
  c.n = geom.n;
  c.layers.assign(layers, kicked_ising_layer(geom, theta_x, theta_zz));
  return c;
}

// ------------------------------------------------------------ partition
uint32_t PartitionSpec::default_block_size(uint32_t workers) {
  uint32_t k = 1;
  while ((uint64_t{1} << k) < workers) ++k;
  return k;
}
PartitionSpec PartitionSpec::make(uint32_t workers, uint32_t k, uint32_t s) {
  if (workers < 1) throw std::invalid_argument("worker_count must be >= 1");
  if (k < 1 || k > 32) throw std::invalid_argument("block_size_bits must be in [1, 32]");
  if (s < 1) throw std::invalid_argument("perturbation_s must be >= 1");
  return PartitionSpec{workers, k, s};
}
// Block-sum owner map, paper Eq. 9 (partition.cpp:53-59).
uint32_t owner(const PartitionSpec& spec, const PauliString& index, int n) {
  const uint32_t k = spec.block_size_bits;
  const uint32_t blocks = (2 * (uint32_t)n + k - 1) / k;
  uint64_t sum = 0;
  for (uint32_t j = 0; j < blocks; ++j) {
    uint64_t lo = (uint64_t)j * k;
    size_t w = lo >> 6;
    if (w >= index.words.size()) continue;
    int sh = (int)(lo & 63);
    uint64_t v = index.words[w] >> sh;
    if (sh + (int)k > 64 && w + 1 < index.words.size()) v |= index.words[w + 1] << (64 - sh);
    sum += v & ((uint64_t{1} << k) - 1);
  }
  if (spec.perturbation_s > 1) sum += hash_string(index) % spec.perturbation_s;
  return (uint32_t)(sum % spec.worker_count);
}
double uniformity_ratio(const std::vector<size_t>& sizes) {
  if (sizes.empty()) throw std::invalid_argument("uniformity_ratio needs at least one shard");
  auto [lo, hi] = std::minmax_element(sizes.begin(), sizes.end());
  if (*lo == 0) return std::numeric_limits<double>::infinity();
  return double(*hi) / double(*lo);
}

// ------------------------------------------------------------ ledger
const char* RunLedger::csv_header() {
  return "t,observable,term_count,global_max,removed,wall_ms_per_gate,batches_sent,records_sent";
}
std::string RunLedger::csv_row(const LayerRecord& r) {
  char buf[256];
  std::snprintf(buf, sizeof(buf), "%d,%.17g,%llu,%.17g,%llu,%.6g,%llu,%llu", r.t, r.observable,
                (unsigned long long)r.term_count, r.global_max, (unsigned long long)r.removed, r.wall_ms_per_gate,
                (unsigned long long)r.batches_sent, (unsigned long long)r.records_sent);
  return buf;
}
std::string RunLedger::to_csv() const {
  std::ostringstream out;
  out << csv_header() << '\n';
  for (const auto& r : rows) out << csv_row(r) << '\n';
  return out.str();
}

double SparseOperator::coefficient(const PauliString& index) const {
  auto cmp = [](const PauliString& a, const PauliString& b) {
    for (int k = kIndexWords - 1; k >= 0; --k)
      if (a.words[k] != b.words[k]) return a.words[k] < b.words[k];
    return false;
  };
  auto it = std::lower_bound(keys.begin(), keys.end(), index, cmp);
  return (it != keys.end() && *it == index) ? values[it - keys.begin()] : 0.0;
}
double SparseOperator::expectation_zero_state() const {
  double s = 0.0;
  for (size_t i = 0; i < keys.size(); ++i) {
    uint64_t acc = 0;
    for (uint64_t w : keys[i].words) acc |= (w ^ (w >> 1)) & 0x5555555555555555ULL;
    if (!acc) s += values[i];
  }
  return s;
}

// ------------------------------------------------------------ engine
static pp_gate to_pp(const Gate& g) {
  pp_gate p;
  for (int k = 0; k < 4; ++k) p.words[k] = g.generator.words[k];
  p.theta = g.theta;
  p.cos_theta = g.cos_theta;
  p.sin_theta = g.sin_theta;
  return p;
}

void Engine::check(int rc) const {
  if (rc == PP_OK) return;
  std::string msg = pp_last_error(handle_);
  switch (rc) {
    case PP_ERR_INVALID: throw std::invalid_argument(msg);
    case PP_ERR_NUMERICAL: throw NumericalError(msg);
    case PP_ERR_RESOURCE: throw ResourceLimitError(msg);
    default: throw std::runtime_error(msg);
  }
}

Engine::Engine(const EngineConfig& config) : config_(config) {
  if (config.n < 1 || config.n > kMaxQubits) throw std::invalid_argument("qubit count out of range");
  PartitionSpec::make(config.partition.worker_count, config.partition.block_size_bits, config.partition.perturbation_s);
  if (config.policy.epsilon0 < 0) throw std::invalid_argument("epsilon0 must be >= 0");
  pp_config c{};
  c.n = config.n;
  c.epsilon0 = config.policy.epsilon0;
  c.cadence = config.policy.cadence == TruncationCadence::PerLayer ? PP_CADENCE_LAYER : PP_CADENCE_GATE;
  c.max_terms = config.max_terms;
  c.workers = config.partition.worker_count;
  c.device = config.device;
  c.flags = (config.fuse_clifford ? 0u : PP_FLAG_NO_CLIFFORD_FUSION) | (config.profile ? PP_FLAG_PROFILE : 0u) |
            (config.external_truncation ? PP_FLAG_EXTERNAL_TRUNCATION : 0u);
  c.mem_fraction = 0.0;
  int rc = pp_create(&c, &handle_);
  if (rc != PP_OK) {
    std::string msg = pp_last_error(nullptr);
    if (rc == PP_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
}
Engine::~Engine() {
  if (handle_) pp_destroy(handle_);
}
Engine::Engine(Engine&& o) noexcept : config_(o.config_), handle_(o.handle_), layer_context_(o.layer_context_) {
  o.handle_ = nullptr;
}
Engine& Engine::operator=(Engine&& o) noexcept {
  if (this != &o) {
    if (handle_) pp_destroy(handle_);
    config_ = o.config_;
    handle_ = o.handle_;
    layer_context_ = o.layer_context_;
    o.handle_ = nullptr;
  }
  return *this;
}

void Engine::set_initial(const std::vector<std::pair<PauliString, double>>& terms) {
  std::vector<uint64_t> w(4 * terms.size());
  std::vector<double> c(terms.size());
  for (size_t i = 0; i < terms.size(); ++i) {
    for (int k = 0; k < 4; ++k) w[4 * i + k] = terms[i].first.words[k];
    c[i] = terms[i].second;
  }
  check(pp_set_initial(handle_, w.data(), c.data(), terms.size()));
}
void Engine::apply_gate(const Gate& gate) {
  pp_gate g = to_pp(gate);
  check(pp_apply_gate(handle_, &g));
}
void Engine::apply_gates(const std::vector<Gate>& gates) {
  std::vector<pp_gate> g(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) g[i] = to_pp(gates[i]);
  check(pp_apply_gates(handle_, g.data(), g.size()));
}
double Engine::apply_layer(const std::vector<Gate>& gates) {
  std::vector<pp_gate> g(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) g[i] = to_pp(gates[i]);
  double obs = 0.0;
  check(pp_apply_layer(handle_, g.data(), g.size(), &obs));
  return obs;
}
void Engine::truncate_now() { check(pp_truncate_now(handle_)); }
uint64_t Engine::term_count() const {
  uint64_t n = 0;
  check(pp_term_count(handle_, &n));
  return n;
}
double Engine::global_max() const {
  double v = 0;
  check(pp_global_max(handle_, &v));
  return v;
}
double Engine::expectation_zero_state() const {
  double v = 0;
  check(pp_expectation_zero_state(handle_, &v));
  return v;
}
double Engine::coefficient(const PauliString& index) const {
  double v = 0;
  check(pp_coefficient(handle_, index.words.data(), &v));
  return v;
}
SparseOperator Engine::merged() const {
  SparseOperator op;
  op.n = config_.n;
  uint64_t n = term_count(), got = 0;
  std::vector<uint64_t> w(4 * std::max<uint64_t>(n, 1));
  op.values.resize(std::max<uint64_t>(n, 1));
  check(pp_export(handle_, w.data(), op.values.data(), n, &got));
  op.values.resize(got);
  op.keys.resize(got);
  for (uint64_t i = 0; i < got; ++i)
    for (int k = 0; k < 4; ++k) op.keys[i].words[k] = w[4 * i + k];
  return op;
}
Engine::Counters Engine::take_counters() {
  pp_counters c{};
  check(pp_take_counters(handle_, &c));
  Counters out;
  out.removed = c.removed;
  out.batches_sent = c.batches_sent;
  out.records_sent = c.records_sent;
  out.gates = c.gates;
  out.total_ns = c.branch_ns + c.exchange_ns + c.truncate_ns + c.other_ns;
  return out;
}

RunLedger run_circuit(Engine& engine, const Circuit& circuit, const RunOptions& options) {
  if (circuit.n != engine.num_qubits())
    throw std::invalid_argument("circuit width " + std::to_string(circuit.n) + " does not match engine width " +
                                std::to_string(engine.num_qubits()));
  if (circuit.layers.empty()) throw std::invalid_argument("circuit has no layers");
  auto read = [&]() {
    return options.readout == ReadoutMode::ZeroState ? engine.expectation_zero_state()
                                                     : engine.coefficient(options.tracked_index);
  };
  RunLedger ledger;
  const int L = (int)circuit.layers.size();
  engine.take_counters();
  if (options.start_layer < 0 || options.start_layer > L)
    throw std::invalid_argument("start_layer " + std::to_string(options.start_layer) + " outside [0, " +
                                std::to_string(L) + "]");
  for (int t = options.start_layer + 1; t <= L; ++t) {
    engine.set_layer_context(t);
    const auto& layer = circuit.layers[L - t];
    auto t0 = std::chrono::steady_clock::now();
    double fused = 0.0;
    bool have_fused = false;
    if (options.on_gate_readout) {
      size_t gi = 0;
      for (auto g = layer.rbegin(); g != layer.rend(); ++g, ++gi) {
        engine.apply_gate(*g);
        options.on_gate_readout(t, gi, read());
      }
    } else {
      std::vector<Gate> rev(layer.rbegin(), layer.rend());
      if (options.readout == ReadoutMode::ZeroState &&
          engine.config().policy.cadence == TruncationCadence::PerGate) {
        fused = engine.apply_layer(rev);  // gates + readout in one device round trip
        have_fused = true;
      } else {
        engine.apply_gates(rev);
      }
    }
    if (engine.config().policy.cadence == TruncationCadence::PerLayer) engine.truncate_now();
    double wall_ns =
        (double)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    Engine::Counters c = engine.take_counters();
    LayerRecord row;
    row.t = t;
    row.observable = have_fused ? fused : read();
    row.term_count = engine.term_count();
    row.global_max = engine.global_max();
    row.removed = c.removed;
    row.wall_ms_per_gate = c.gates ? 1e-6 * wall_ns / double(c.gates) : 0.0;
    row.batches_sent = c.batches_sent;
    row.records_sent = c.records_sent;
    ledger.rows.push_back(row);
    if (options.on_layer) options.on_layer(row, engine);
  }
  return ledger;
}

// ------------------------------------------------------------ diagnostics and checkpoints
static std::string fmt17(double v) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

DensityHistogram histogram_from_counts(int bins, double epsilon0, const std::vector<uint64_t>& pos,
                                       const std::vector<uint64_t>& neg) {
  if (bins < 1) throw std::invalid_argument("histogram needs at least 1 bin");
  if ((int)pos.size() != bins || (int)neg.size() != bins) throw std::invalid_argument("histogram count size");
  DensityHistogram h;
  const double lower = std::max(epsilon0, 1e-16);
  const double log_lower = std::log(lower);
  h.bin_edges.resize(bins + 1);
  for (int b = 0; b <= bins; ++b) h.bin_edges[b] = std::exp(log_lower * (1.0 - double(b) / bins));
  h.bin_edges[bins] = 1.0;
  h.positive.assign(bins, 0.0);
  h.negative.assign(bins, 0.0);
  h.positive_counts = pos;
  h.negative_counts = neg;
  uint64_t total = 0;
  for (int b = 0; b < bins; ++b) total += pos[b] + neg[b];
  h.total_terms = total;
  if (total == 0) return h;
  const double inv_norm = 1.0 / double(total);
  // same sequence of roundings as the reference's per-string accumulation
  for (int b = 0; b < bins; ++b) {
    double sp = 0.0, sn = 0.0;
    for (uint64_t k = 0; k < pos[b]; ++k) sp += inv_norm;
    for (uint64_t k = 0; k < neg[b]; ++k) sn += inv_norm;
    h.positive[b] = sp;
    h.negative[b] = sn;
  }
  return h;
}

DensityHistogram density_histogram(const Engine& engine, int bins, double epsilon0, double global_max) {
  if (bins < 1) throw std::invalid_argument("histogram needs at least 1 bin");
  std::vector<uint64_t> pos(bins), neg(bins);
  engine.check(pp_density_histogram(engine.handle(), bins, global_max, epsilon0, pos.data(), neg.data()));
  return histogram_from_counts(bins, epsilon0, pos, neg);
}
DensityHistogram density_histogram(const Engine& engine, int bins, double epsilon0) {
  return density_histogram(engine, bins, epsilon0, engine.global_max());
}

std::string DensityHistogram::to_tsv() const {
  std::ostringstream out;
  out << "bin_low\tbin_high\tsign\tnormalized_count\n";
  for (size_t b = 0; b + 1 < bin_edges.size(); ++b) {
    out << fmt17(bin_edges[b]) << '\t' << fmt17(bin_edges[b + 1]) << "\t+\t" << fmt17(positive[b]) << '\n';
    out << fmt17(bin_edges[b]) << '\t' << fmt17(bin_edges[b + 1]) << "\t-\t" << fmt17(negative[b]) << '\n';
  }
  return out.str();
}

void dump_operator(std::ostream& out, const SparseOperator& op) {
  for (size_t i = 0; i < op.keys.size(); ++i) out << to_hex(op.keys[i], op.n) << ' ' << fmt17(op.values[i]) << '\n';
}

static void sort_operator(SparseOperator& op) {
  std::vector<size_t> idx(op.keys.size());
  for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
  auto less = [&](size_t a, size_t b) {
    for (int k = kIndexWords - 1; k >= 0; --k)
      if (op.keys[a].words[k] != op.keys[b].words[k]) return op.keys[a].words[k] < op.keys[b].words[k];
    return false;
  };
  std::sort(idx.begin(), idx.end(), less);
  SparseOperator out;
  out.n = op.n;
  for (size_t i : idx) {
    if (!out.keys.empty() && out.keys.back() == op.keys[i]) {
      out.values.back() += op.values[i];
      continue;
    }
    out.keys.push_back(op.keys[i]);
    out.values.push_back(op.values[i]);
  }
  op = std::move(out);
}

SparseOperator load_dump(std::istream& in, int n) {
  SparseOperator op;
  op.n = n;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ls(line);
    std::string hex;
    double value;
    if (!(ls >> hex >> value)) throw std::invalid_argument("malformed dump line: " + line);
    op.keys.push_back(from_hex(hex, n));
    op.values.push_back(value);
  }
  sort_operator(op);
  return op;
}

static const char kBinMagic[4] = {'P', 'P', 'B', '1'};

void write_shard_file(const std::string& path, const SparseOperator& op, bool binary) {
  std::ofstream out(path, binary ? std::ios::binary : std::ios::out);
  if (!out) throw std::runtime_error("cannot write " + path);
  if (!binary) {
    dump_operator(out, op);
  } else {
    const uint32_t n = (uint32_t)op.n;
    const uint64_t count = op.keys.size();
    out.write(kBinMagic, 4);
    out.write(reinterpret_cast<const char*>(&n), 4);
    out.write(reinterpret_cast<const char*>(&count), 8);
    for (const auto& k : op.keys) out.write(reinterpret_cast<const char*>(k.words.data()), 8 * kIndexWords);
    out.write(reinterpret_cast<const char*>(op.values.data()), 8 * count);
  }
  if (!out) throw std::runtime_error("write failed: " + path);
}

static SparseOperator read_shard_file(const std::string& path, int n) {
  const bool binary = path.size() > 4 && path.compare(path.size() - 4, 4, ".ppb") == 0;
  std::ifstream in(path, binary ? std::ios::binary : std::ios::in);
  if (!in) throw std::invalid_argument("cannot open checkpoint shard " + path);
  if (!binary) return load_dump(in, n);
  char magic[4];
  uint32_t fn = 0;
  uint64_t count = 0;
  in.read(magic, 4);
  in.read(reinterpret_cast<char*>(&fn), 4);
  in.read(reinterpret_cast<char*>(&count), 8);
  if (!in || std::memcmp(magic, kBinMagic, 4) != 0) throw std::invalid_argument("not a binary shard: " + path);
  if ((int)fn != n) throw std::invalid_argument("shard " + path + " width does not match the manifest");
  SparseOperator op;
  op.n = n;
  op.keys.resize(count);
  op.values.resize(count);
  for (auto& k : op.keys) in.read(reinterpret_cast<char*>(k.words.data()), 8 * kIndexWords);
  in.read(reinterpret_cast<char*>(op.values.data()), 8 * count);
  if (!in) throw std::invalid_argument("truncated binary shard " + path);
  sort_operator(op);
  return op;
}

void write_checkpoint_manifest(const std::string& dir, int layer, int qubits, double epsilon0,
                               const std::vector<std::pair<std::string, uint64_t>>& files) {
  std::ofstream mf(dir + "/manifest.json");
  if (!mf) throw std::runtime_error("cannot write " + dir + "/manifest.json");
  mf << "{\n  \"schema\": 1,\n  \"layer\": " << layer << ",\n  \"qubits\": " << qubits
     << ",\n  \"workers\": " << files.size() << ",\n  \"epsilon0\": " << fmt17(epsilon0)
     << ",\n  \"shard_map\": \"z-plane splitmix hash\",\n  \"files\": [";
  for (size_t m = 0; m < files.size(); ++m) {
    mf << (m ? "," : "") << "\n    {\n      \"path\": \"" << files[m].first << "\",\n      \"terms\": "
       << files[m].second << ",\n      \"worker\": " << m << "\n    }";
  }
  mf << "\n  ]\n}\n";
}

void write_checkpoint(const std::string& dir, const Engine& engine, int layer, bool binary) {
  for (size_t i = 1; i <= dir.size(); ++i)  // mkdir -p (fs::create_directories in runner.cpp:54)
    if (i == dir.size() || dir[i] == '/') ::mkdir(dir.substr(0, i).c_str(), 0777);
  SparseOperator op = engine.merged();
  const std::string name = binary ? "shard_0.ppb" : "shard_0.txt";
  write_shard_file(dir + "/" + name, op, binary);
  write_checkpoint_manifest(dir, layer, engine.num_qubits(), engine.config().policy.epsilon0,
                            {{name, (uint64_t)op.keys.size()}});
}

// minimal reader for the manifest keys we need (nlohmann's dump(2) layout and ours)
static bool json_number(const std::string& text, const std::string& key, double* out) {
  size_t p = text.find("\"" + key + "\"");
  if (p == std::string::npos) return false;
  p = text.find(':', p);
  if (p == std::string::npos) return false;
  *out = std::strtod(text.c_str() + p + 1, nullptr);
  return true;
}

Checkpoint read_checkpoint(const std::string& dir) {
  std::ifstream mf(dir + "/manifest.json");
  if (!mf) throw std::invalid_argument("no manifest.json in " + dir);
  std::string text((std::istreambuf_iterator<char>(mf)), std::istreambuf_iterator<char>());
  Checkpoint ck;
  double v = 0;
  if (!json_number(text, "layer", &v)) throw std::invalid_argument("manifest has no layer");
  ck.layer = (int)v;
  if (!json_number(text, "qubits", &v)) throw std::invalid_argument("manifest has no qubits");
  ck.qubits = (int)v;
  if (json_number(text, "epsilon0", &v)) ck.epsilon0 = v;
  ck.op.n = ck.qubits;
  std::vector<std::string> paths;
  for (size_t p = text.find("\"path\""); p != std::string::npos; p = text.find("\"path\"", p + 6)) {
    size_t a = text.find('"', text.find(':', p) + 1);
    size_t b = text.find('"', a + 1);
    if (a == std::string::npos || b == std::string::npos) throw std::invalid_argument("malformed manifest");
    paths.push_back(text.substr(a + 1, b - a - 1));
  }
  if (paths.empty()) throw std::invalid_argument("manifest lists no shard files");
  for (const auto& name : paths) {
    SparseOperator part = read_shard_file(dir + "/" + name, ck.qubits);
    ck.op.keys.insert(ck.op.keys.end(), part.keys.begin(), part.keys.end());
    ck.op.values.insert(ck.op.values.end(), part.values.begin(), part.values.end());
  }
  sort_operator(ck.op);
  return ck;
}

}  // namespace pauliprop
