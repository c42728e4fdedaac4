// pauliprop.cpp -- host side of the B200 engine: Pauli-string algebra and
// I/O, angles and circuits, geometries and the kicked-Ising builder, and the
// Engine / run_circuit front end over the C-ABI (include/pauliprop_gpu.h).
//
// Behaviour follows the reference API it stands in for; each block cites the
// reference function whose contract it keeps.
#include "pauliprop.hpp"

#include <algorithm>
#include <cerrno>
#include <charconv>
#include <climits>
#include <numeric>
#include <string_view>
#include <utility>
#include <chrono>
#include <cmath>
#include <complex>
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
constexpr char kLetters[] = "IXYZ";
constexpr char kHexDigits[] = "0123456789abcdef";
constexpr uint64_t kEven = 0x5555555555555555ULL;

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
  const char* p = std::strchr(kLetters, c);
  return (p && c) ? int(p - kLetters) : -1;
}

int hex_value(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

bool is_blank(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

// x/z bit planes of one packed word (site s at bits 2s, 2s+1 -> plane bit 2s):
// X = (x, !z), Y = (x, z), Z = (!x, z).
struct Planes {
  uint64_t x, z;
};
Planes planes_of(uint64_t w) {
  const uint64_t lo = w & kEven, hi = (w >> 1) & kEven;
  return {lo ^ hi, hi};
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

// sigma_a sigma_b = i^{local_phase(a, b)} sigma_{a xor b} on one site
// (pauli_string.cpp:25-34): +1 for the cyclic pairs XY, YZ, ZX, -1 for the
// reversed ones, 0 when either is I or a == b.
int local_phase(uint8_t a, uint8_t b) {
  a &= 3, b &= 3;
  if (!a || !b || a == b) return 0;
  return b == a % 3 + 1 ? 1 : -1;
}

// B(I, J) mod 4 (pauli_string.cpp:79-85) from bit planes: the number of
// cyclic site pairs minus the number of anti-cyclic ones.
int phase_exponent(const PauliString& I, const PauliString& J, int n) {
  int b = 0;
  for (int w = 0; w < kIndexWords && 32 * w < n; ++w) {
    uint64_t keep = kEven;
    if (n - 32 * w < 32) keep &= (uint64_t{1} << (2 * (n - 32 * w))) - 1;
    const Planes p = planes_of(I.words[w]), q = planes_of(J.words[w]);
    const uint64_t pX = p.x & ~p.z & keep, pY = p.x & p.z & keep, pZ = ~p.x & p.z & keep;
    const uint64_t qX = q.x & ~q.z, qY = q.x & q.z, qZ = ~q.x & q.z;
    b += __builtin_popcountll((pX & qY) | (pY & qZ) | (pZ & qX));
    b -= __builtin_popcountll((pY & qX) | (pZ & qY) | (pX & qZ));
  }
  return ((b % 4) + 4) % 4;
}

bool commutes(const PauliString& I, const PauliString& J, int n) { return (phase_exponent(I, J, n) & 1) == 0; }

StringProduct string_product(const PauliString& I, const PauliString& J, int n) {
  return {I ^ J, phase_exponent(I, J, n)};
}

int pauli_weight(const PauliString& s) {
  int w = 0;
  for (uint64_t v : s.words) w += __builtin_popcountll((v | (v >> 1)) & kEven);
  return w;
}

// ------------------------------------------------------------ text helpers
// A line-oriented view of a text block: '#' starts a comment, tokens are
// separated by blanks/tabs/CR.  Shared by the circuit and geometry readers.
namespace {
struct TextLine {
  int number = 0;
  std::vector<std::string_view> tokens;
};

std::vector<std::string_view> split_tokens(std::string_view text) {
  std::vector<std::string_view> tokens;
  size_t p = 0;
  while (p < text.size()) {
    while (p < text.size() && is_blank(text[p])) ++p;
    size_t q = p;
    while (q < text.size() && !is_blank(text[q])) ++q;
    if (q > p) tokens.push_back(text.substr(p, q - p));
    p = q;
  }
  return tokens;
}

std::vector<TextLine> split_lines(std::string_view text) {
  std::vector<TextLine> out;
  int number = 0;
  while (!text.empty() || number == 0) {
    size_t eol = text.find('\n');
    std::string_view raw = text.substr(0, eol);
    text = eol == std::string_view::npos ? std::string_view{} : text.substr(eol + 1);
    TextLine tl;
    tl.number = ++number;
    tl.tokens = split_tokens(raw.substr(0, raw.find('#')));
    out.push_back(std::move(tl));
    if (eol == std::string_view::npos) break;
  }
  return out;
}

[[noreturn]] void line_error(const char* what, int number, const std::string& msg) {
  throw std::invalid_argument(std::string(what) + " line " + std::to_string(number) + ": " + msg);
}

// Whole-token integer; false if the token has anything else in it.
bool token_int(std::string_view tok, long long* out) {
  if (tok.empty()) return false;
  const char* first = tok.data();
  if (*first == '+') ++first;  // operator>> accepts an explicit plus
  auto [end, ec] = std::from_chars(first, tok.data() + tok.size(), *out);
  return ec == std::errc() && end == tok.data() + tok.size();
}

// Leading integer of a token, as operator>> would extract it (rest ignored).
bool leading_int(std::string_view tok, long long* out) {
  const char* first = tok.data();
  if (!tok.empty() && *first == '+') ++first;
  auto [end, ec] = std::from_chars(first, tok.data() + tok.size(), *out);
  return ec == std::errc() && end != first;
}
}  // namespace

// ------------------------------------------------------------ labels
// Two label forms (pauli_string.cpp:105-177): dense, one letter per site with
// the leftmost letter = site n-1; sparse, blank-separated "<P><site>" tokens.
// A label containing a digit or a blank is sparse.
PauliString parse_pauli_label(const std::string& text, int n) {
  if (n < 1 || n > kMaxQubits) throw std::invalid_argument("qubit count out of range: " + std::to_string(n));
  std::string_view body = text;
  while (!body.empty() && (body.front() == ' ' || body.front() == '\t')) body.remove_prefix(1);
  while (!body.empty() && (body.back() == ' ' || body.back() == '\t')) body.remove_suffix(1);
  if (body.empty()) throw std::invalid_argument("empty pauli label");
  const bool sparse = std::any_of(body.begin(), body.end(),
                                  [](char ch) { return is_blank(ch) || (ch >= '0' && ch <= '9'); });
  PauliString s;
  if (!sparse) {
    if ((int)body.size() != n)
      throw std::invalid_argument("dense pauli label \"" + std::string(body) + "\" has length " +
                                  std::to_string(body.size()) + ", expected n=" + std::to_string(n));
    int site = n;
    for (char ch : body) {
      --site;
      const int code = code_of(ch);
      if (code < 0) throw std::invalid_argument(std::string("invalid pauli character '") + ch + "'");
      s.set_code(site, (uint8_t)code);
    }
    return s;
  }
  {
    for (std::string_view tok : split_tokens(body)) {
      const std::string t(tok);
      const int code = code_of(tok[0]);
      if (code <= 0) throw std::invalid_argument("invalid sparse pauli token \"" + t + "\"");
      if (tok.size() == 1) throw std::invalid_argument("sparse pauli token \"" + t + "\" is missing a site index");
      long long site = 0;
      std::string_view digits = tok.substr(1);
      // std::stoi semantics: leading blanks/sign allowed, then digits; the
      // whole remainder must be consumed
      const char* b = digits.data();
      const char* e = b + digits.size();
      const char* num = (*b == '+') ? b + 1 : b;
      auto [end, ec] = std::from_chars(num, e, site);
      if (ec != std::errc() || end == num || site < INT_MIN || site > INT_MAX)
        throw std::invalid_argument("invalid site index in token \"" + t + "\"");
      if (end != e) throw std::invalid_argument("invalid sparse pauli token \"" + t + "\"");
      require_site((int)site, n);
      if (s.code_at((int)site) != 0)
        throw std::invalid_argument("site " + std::to_string(site) + " appears twice in pauli label");
      s.set_code((int)site, (uint8_t)code);
    }
  }
  return s;
}

std::string to_dense_label(const PauliString& s, int n) {
  std::string out;
  out.reserve(n);
  for (int site = n - 1; site >= 0; --site) out.push_back(kLetters[s.code_at(site)]);
  return out;
}

std::string to_sparse_label(const PauliString& s, int n) {
  std::ostringstream out;
  const char* sep = "";
  for (int site = 0; site < n; ++site) {
    if (uint8_t c = s.code_at(site)) {
      out << sep << kLetters[c] << site;
      sep = " ";
    }
  }
  std::string r = out.str();
  return r.empty() ? std::string("I") : r;
}

// Hex index (checkpoint dumps, sparse_operator.cpp:99-122): 2n bits, most
// significant nibble first, ceil(2n/4) digits.
std::string to_hex(const PauliString& s, int n) {
  const int nibbles = (2 * n + 3) / 4;
  std::string out;
  out.reserve(nibbles);
  for (int d = nibbles - 1; d >= 0; --d) {
    const uint64_t word = s.words[(4 * d) / 64];
    out.push_back(kHexDigits[(word >> ((4 * d) % 64)) & 0xFu]);
  }
  return out;
}

PauliString from_hex(const std::string& hex, int n) {
  PauliString s;
  const int len = (int)hex.size();
  for (int d = 0; d < len; ++d) {  // d = nibble index from the least significant end
    const char ch = hex[len - 1 - d];
    const int v = hex_value(ch);
    if (v < 0) throw std::invalid_argument(std::string("invalid hex digit '") + ch + "'");
    if (v == 0) continue;
    if (4 * d >= 2 * kMaxQubits) throw std::invalid_argument("hex index wider than the maximum width");
    s.words[(4 * d) / 64] |= uint64_t(v) << ((4 * d) % 64);
  }
  // every code above site n-1 must be identity
  for (int w = 0; w < kIndexWords; ++w) {
    const int lo_site = 32 * w;
    uint64_t allowed = 0;
    if (n >= lo_site + 32) allowed = ~uint64_t{0};
    else if (n > lo_site) allowed = (uint64_t{1} << (2 * (n - lo_site))) - 1;
    if (s.words[w] & ~allowed) throw std::invalid_argument("hex index has bits above site " + std::to_string(n - 1));
  }
  return s;
}

// ------------------------------------------------------------ angles
// Exact trig at half-integer multiples of pi (circuit.cpp:28-40): the
// quarter-turn grid is looked up, everything else goes to libm.
static double cos_pi(double r) {
  double f = std::fmod(r, 2.0);
  if (f < 0) f += 2.0;
  const double quarter = 2.0 * f;
  if (quarter == std::floor(quarter)) {
    static constexpr double kGrid[4] = {1.0, 0.0, -1.0, 0.0};
    return kGrid[static_cast<int>(quarter) & 3];
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

// "<number>" radians or "<number>pi" / "pi" / "-pi" pi units (circuit.cpp:65-87).
Angle parse_angle(const std::string& text) {
  std::string number = text;
  const bool pi_units = text.size() >= 2 && (text.compare(text.size() - 2, 2, "pi") == 0 ||
                                             text.compare(text.size() - 2, 2, "PI") == 0);
  if (pi_units) {
    number.resize(number.size() - 2);
    if (number.empty() || number == "+" || number == "-") number.push_back('1');  // "pi", "-pi"
  }
  const char* begin = number.c_str();
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(begin, &end);
  if (end == begin || *end != '\0' || errno == ERANGE) throw std::invalid_argument("invalid angle \"" + text + "\"");
  if (!std::isfinite(v)) throw std::invalid_argument("angle must be finite: \"" + text + "\"");
  return pi_units ? Angle::from_pi_units(v) : Angle::from_radians(v);
}

Gate::Gate(const PauliString& g, Angle a)
    : generator(g), theta(a.radians), cos_theta(a.cosine()), sin_theta(a.sine()) {}

size_t Circuit::total_gates() const {
  return std::accumulate(layers.begin(), layers.end(), size_t{0},
                         [](size_t acc, const std::vector<Gate>& l) { return acc + l.size(); });
}

// Circuit text (circuit.cpp:101-137): one "<label> <angle>" gate per line;
// the angle is the last token, everything before it is the label; blank
// (or comment-only) lines close the current layer.
Circuit parse_circuit_text(const std::string& text, int n) {
  Circuit c;
  c.n = n;
  std::vector<Gate> open;
  auto close_layer = [&] {
    if (!open.empty()) c.layers.push_back(std::exchange(open, {}));
  };
  for (const TextLine& tl : split_lines(text)) {
    if (tl.tokens.empty()) {
      close_layer();
      continue;
    }
    if (tl.tokens.size() < 2) line_error("circuit", tl.number, "expected \"pauli-label angle\"");
    std::string label;
    for (size_t k = 0; k + 1 < tl.tokens.size(); ++k) {
      if (k) label.push_back(' ');
      label.append(tl.tokens[k]);
    }
    try {
      open.emplace_back(parse_pauli_label(label, n), parse_angle(std::string(tl.tokens.back())));
    } catch (const std::invalid_argument& e) {
      line_error("circuit", tl.number, e.what());
    }
  }
  close_layer();
  return c;
}

std::string format_circuit(const Circuit& c) {
  std::string out;
  char theta[40];
  bool first_layer = true;
  for (const auto& layer : c.layers) {
    if (!first_layer) out.push_back('\n');
    first_layer = false;
    for (const Gate& g : layer) {
      std::snprintf(theta, sizeof(theta), "%.17g", g.theta);
      out += to_sparse_label(g.generator, c.n);
      out.push_back(' ');
      out += theta;
      out.push_back('\n');
    }
  }
  return out;
}

// ------------------------------------------------------------ geometry
// Edge-list text (models.cpp:27-105): "i j" or "i j color" per line, the
// file either fully coloured or not at all, no self loops or repeated
// edges, and each colour class a matching.  A line whose first token is not
// an integer carries no edge.
Geometry load_geometry_text(const std::string& text) {
  struct Row {
    int line, i, j, color;
  };
  std::vector<Row> rows;
  for (const TextLine& tl : split_lines(text)) {
    long long i = 0, j = 0, color = -1;
    if (tl.tokens.empty() || !leading_int(tl.tokens[0], &i)) continue;
    if (!token_int(tl.tokens[0], &i) || tl.tokens.size() < 2 || !leading_int(tl.tokens[1], &j))
      line_error("geometry", tl.number, "expected \"i j [color]\"");
    if (!token_int(tl.tokens[1], &j))
      line_error("geometry", tl.number, "expected \"i j [color]\"");
    size_t used = 2;
    if (tl.tokens.size() > 2 && token_int(tl.tokens[2], &color)) {
      if (color < 0) line_error("geometry", tl.number, "negative color");
      used = 3;
    }
    if (tl.tokens.size() > used)
      line_error("geometry", tl.number, "trailing content \"" + std::string(tl.tokens[used]) + "\"");
    if (i < 0 || j < 0) line_error("geometry", tl.number, "negative qubit index");
    if (i == j) line_error("geometry", tl.number, "self loop on qubit " + std::to_string(i));
    rows.push_back({tl.number, (int)i, (int)j, (int)color});
  }
  if (rows.empty()) throw std::invalid_argument("geometry file has no edges");

  Geometry g;
  std::set<std::pair<int, int>> undirected;
  for (const Row& r : rows) {
    if (!undirected.emplace(std::min(r.i, r.j), std::max(r.i, r.j)).second)
      line_error("geometry", r.line, "duplicate edge " + std::to_string(r.i) + "-" + std::to_string(r.j));
    g.edges.emplace_back(r.i, r.j);
    g.edge_colors.push_back(r.color);
    g.n = std::max(g.n, std::max(r.i, r.j) + 1);
  }
  const size_t coloured = (size_t)std::count_if(rows.begin(), rows.end(), [](const Row& r) { return r.color >= 0; });
  if (coloured != 0 && coloured != rows.size())
    throw std::invalid_argument("geometry file mixes colored and uncolored edges");
  if (coloured == 0) {
    g.edge_colors.clear();
    return g;
  }
  g.color_count = 1 + *std::max_element(g.edge_colors.begin(), g.edge_colors.end());
  // (qubit, colour) pairs must be unique: every colour class is a matching
  std::set<std::pair<int, int>> incident;
  for (size_t e = 0; e < g.edges.size(); ++e) {
    const int col = g.edge_colors[e];
    if (!incident.emplace(g.edges[e].first, col).second || !incident.emplace(g.edges[e].second, col).second)
      throw std::invalid_argument("edges overlap within color " + std::to_string(col) + " at edge " +
                                  std::to_string(g.edges[e].first) + "-" + std::to_string(g.edges[e].second));
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

#include "heavy_hex_127.inc"

// The reference's bundled 127-qubit heavy-hex map, same edges, colours and
// edge order (models.cpp:120 loads data/heavy_hex_127.txt through
// heavy_hex_data.cpp:21), so build_kicked_ising produces the reference's gate
// order.  It equals the BASELINE.json config-1 row/bridge construction.
Geometry heavy_hex_127() {
  Geometry g;
  g.n = 127;
  g.color_count = 3;
  for (const auto& e : kHeavyHex127) {
    g.edges.emplace_back(e[0], e[1]);
    g.edge_colors.push_back(e[2]);
  }
  return g;
}

// Qubits within graph distance `radius` of `start`, ascending
// (models.cpp:122-147), by frontier expansion over a CSR adjacency.
std::vector<int> bfs_ball(const Geometry& geom, int start, int radius) {
  std::vector<int> offset(geom.n + 1, 0), nbr(2 * geom.edges.size());
  for (auto [a, b] : geom.edges) ++offset[a + 1], ++offset[b + 1];
  std::partial_sum(offset.begin(), offset.end(), offset.begin());
  std::vector<int> fill(offset.begin(), offset.end() - 1);
  for (auto [a, b] : geom.edges) nbr[fill[a]++] = b, nbr[fill[b]++] = a;
  std::vector<char> in_ball(geom.n, 0);
  std::vector<int> frontier{start}, next;
  in_ball[start] = 1;
  for (int d = 0; d < radius && !frontier.empty(); ++d) {
    next.clear();
    for (int u : frontier)
      for (int k = offset[u]; k < offset[u + 1]; ++k)
        if (!in_ball[nbr[k]]) in_ball[nbr[k]] = 1, next.push_back(nbr[k]);
    frontier.swap(next);
  }
  std::vector<int> ball;
  for (int q = 0; q < geom.n; ++q)
    if (in_ball[q]) ball.push_back(q);
  return ball;
}

// One Trotter step (models.cpp:149-171): X on every qubit in index order,
// then the ZZ bonds colour class by colour class, each class in edge-list
// order (a stable sort of the edges by colour).
std::vector<Gate> kicked_ising_layer(const Geometry& geom, Angle theta_x, Angle theta_zz) {
  std::vector<size_t> order(geom.edges.size());
  std::iota(order.begin(), order.end(), size_t{0});
  if (geom.has_coloring())
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t a, size_t b) { return geom.edge_colors[a] < geom.edge_colors[b]; });
  std::vector<Gate> layer;
  layer.reserve(geom.n + order.size());
  for (int q = 0; q < geom.n; ++q) layer.emplace_back(single_site(q, Pauli::X), theta_x);
  for (size_t e : order) {
    const auto [a, b] = geom.edges[e];
    layer.emplace_back(single_site(a, Pauli::Z) ^ single_site(b, Pauli::Z), theta_zz);
  }
  return layer;
}

Circuit build_kicked_ising(const Geometry& geom, Angle theta_x, Angle theta_zz, int layers) {
  if (layers < 1) throw std::invalid_argument("layer count must be >= 1");
  Circuit c;
  c.n = geom.n;
  c.layers = std::vector<std::vector<Gate>>(layers, kicked_ising_layer(geom, theta_x, theta_zz));
  return c;
}

// ------------------------------------------------------------ partition
// The paper's block-sum owner map (partition.cpp:35-59),
// kept for the ledger's worker accounting: owner = (sum over the k-bit blocks
// of the packed 2n-bit index [+ hash % s]) mod workers.  Summing k-bit blocks
// weighs bit i by 2^(i mod k), which is how it is evaluated here.
uint32_t PartitionSpec::default_block_size(uint32_t workers) {
  uint32_t k = 1;
  while (k < 32 && (uint64_t{1} << k) < workers) ++k;
  return k;
}
PartitionSpec PartitionSpec::make(uint32_t workers, uint32_t k, uint32_t s) {
  if (workers < 1) throw std::invalid_argument("worker_count must be >= 1");
  if (k < 1 || k > 32) throw std::invalid_argument("block_size_bits must be in [1, 32]");
  if (s < 1) throw std::invalid_argument("perturbation_s must be >= 1");
  return PartitionSpec{workers, k, s};
}
uint64_t block_sum(const PauliString& index, int n, uint32_t k) {
  const uint32_t span = (2u * (uint32_t)n + k - 1) / k * k;  // whole blocks cover the 2n bits
  uint64_t sum = 0;
  for (int w = 0; w < kIndexWords; ++w) {
    for (uint64_t v = index.words[w]; v; v &= v - 1) {
      const uint32_t bit = 64u * w + (uint32_t)__builtin_ctzll(v);
      if (bit < span) sum += uint64_t{1} << (bit % k);
    }
  }
  return sum;
}
uint32_t owner(const PartitionSpec& spec, const PauliString& index, int n) {
  uint64_t sum = block_sum(index, n, spec.block_size_bits);
  if (spec.perturbation_s > 1) sum += hash_string(index) % spec.perturbation_s;
  return (uint32_t)(sum % spec.worker_count);
}
double uniformity_ratio(const std::vector<size_t>& sizes) {
  if (sizes.empty()) throw std::invalid_argument("uniformity_ratio needs at least one shard");
  const auto [lo, hi] = std::minmax_element(sizes.begin(), sizes.end());
  return *lo == 0 ? std::numeric_limits<double>::infinity() : double(*hi) / double(*lo);
}


std::vector<uint32_t> destination_set(const PartitionSpec& spec, uint32_t m, const PauliString& J, int n) {
  const uint32_t N = spec.worker_count;
  std::vector<uint32_t> out;
  if (spec.perturbation_s > 1) {  // the perturbed map bounds nothing
    for (uint32_t r = 0; r < N; ++r) out.push_back(r);
    return out;
  }
  // XOR-ing a k-bit block j of J into a source block b moves the block sum by
  // jb - 2 (b & jb) for some subset of jb's bits; the residues mod N reachable
  // by summing one such move per block of J are the possible owner shifts.
  const uint32_t k = spec.block_size_bits;
  const uint32_t span = (2u * (uint32_t)n + k - 1) / k * k;
  std::vector<uint64_t> jblocks;
  for (uint32_t lo = 0; lo < span; lo += k) {
    uint64_t v = 0;
    for (uint32_t b = 0; b < k && lo + b < 64u * kIndexWords; ++b)
      v |= ((J.words[(lo + b) / 64] >> ((lo + b) % 64)) & 1u) << b;
    if (v) jblocks.push_back(v);
  }
  std::vector<char> reach(N, 0), next(N);
  reach[0] = 1;
  for (uint64_t jb : jblocks) {
    std::fill(next.begin(), next.end(), 0);
    for (uint64_t sub = jb;; sub = (sub - 1) & jb) {  // every subset of jb's bits
      const int64_t d = (int64_t)jb - 2 * (int64_t)sub;
      const uint32_t dm = (uint32_t)(((d % (int64_t)N) + (int64_t)N) % (int64_t)N);
      for (uint32_t r = 0; r < N; ++r)
        if (reach[r]) next[(r + dm) % N] = 1;
      if (sub == 0) break;
    }
    reach.swap(next);
  }
  for (uint32_t r = 0; r < N; ++r)
    if (reach[r]) out.push_back((m + r) % N);
  std::sort(out.begin(), out.end());
  return out;
}

// ------------------------------------------------------------ dense check
// A Pauli string on the computational basis: P|b> = i^ny (-1)^popc(b & z) |b ^ x>
// with x, z its bit planes (site q -> bit q) and ny its number of Y sites.
namespace {
struct BasisAction {
  uint64_t x = 0, z = 0;
  int ny = 0;
};
BasisAction basis_action(const PauliString& s, int n) {
  BasisAction a;
  for (int q = 0; q < n; ++q) {
    const uint8_t c = s.code_at(q);
    if (c == 1 || c == 2) a.x |= uint64_t{1} << q;
    if (c == 2 || c == 3) a.z |= uint64_t{1} << q;
    if (c == 2) ++a.ny;
  }
  return a;
}
std::complex<double> basis_phase(const BasisAction& a, uint64_t b) {
  static const std::complex<double> ipow[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
  std::complex<double> p = ipow[a.ny & 3];
  return (__builtin_popcountll(b & a.z) & 1) ? -p : p;
}
}  // namespace

double state_vector_expectation(const Circuit& circuit, const PauliString& observable) {
  const int n = circuit.n;
  if (n < 1 || n > 26) throw std::invalid_argument("state_vector_expectation supports 1 <= n <= 26, got " + std::to_string(n));
  std::vector<std::complex<double>> psi(size_t{1} << n);
  psi[0] = 1.0;
  for (const auto& layer : circuit.layers) {
    for (const Gate& g : layer) {  // psi <- (cos(t/2) - i sin(t/2) P) psi, forward in time
      const BasisAction a = basis_action(g.generator, n);
      const std::complex<double> c(std::cos(0.5 * g.theta), 0.0), ms(0.0, -std::sin(0.5 * g.theta));
      for (uint64_t b = 0; b < psi.size(); ++b) {
        const uint64_t p = b ^ a.x;
        if (p < b) continue;
        if (p == b) {  // diagonal generator: a phase per basis state
          psi[b] *= c + ms * basis_phase(a, b);
          continue;
        }
        const std::complex<double> vb = psi[b], vp = psi[p];
        psi[b] = c * vb + ms * basis_phase(a, p) * vp;  // <b|P|p> = phase(p)
        psi[p] = c * vp + ms * basis_phase(a, b) * vb;
      }
    }
  }
  const BasisAction o = basis_action(observable, n);
  std::complex<double> acc = 0.0;
  for (uint64_t b = 0; b < psi.size(); ++b) acc += std::conj(psi[b ^ o.x]) * basis_phase(o, b) * psi[b];
  return acc.real();
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
  // the reference names the layer next to the gate (engine.cpp:269-273,
  // 334-338: "... at layer L, gate G"); the device library knows the gate only
  if (rc == PP_ERR_RESOURCE || rc == PP_ERR_NUMERICAL) {
    const size_t at = msg.find(" at gate ");
    if (at != std::string::npos) msg.replace(at, 9, " at layer " + std::to_string(layer_context_) + ", gate ");
  }
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
    mirror_valid_ = false;
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
  invalidate();
  check(pp_set_initial(handle_, w.data(), c.data(), terms.size()));
}
void Engine::apply_gate(const Gate& gate) {
  invalidate();
  pp_gate g = to_pp(gate);
  check(pp_apply_gate(handle_, &g));
}
void Engine::apply_gates(const std::vector<Gate>& gates) {
  invalidate();
  std::vector<pp_gate> g(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) g[i] = to_pp(gates[i]);
  check(pp_apply_gates(handle_, g.data(), g.size()));
}
double Engine::apply_layer(const std::vector<Gate>& gates) {
  invalidate();
  std::vector<pp_gate> g(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) g[i] = to_pp(gates[i]);
  double obs = 0.0;
  check(pp_apply_layer(handle_, g.data(), g.size(), &obs));
  return obs;
}
void Engine::truncate_now() {
  invalidate();
  check(pp_truncate_now(handle_));
}
std::span<const SparseOperator> Engine::shards() const {
  if (!mirror_valid_) {
    const SparseOperator all = merged();
    const PartitionSpec& spec = config_.partition;
    shard_mirror_.assign(spec.worker_count, SparseOperator{});
    for (auto& sh : shard_mirror_) sh.n = config_.n;
    for (size_t i = 0; i < all.keys.size(); ++i) {  // merged() is sorted: every shard stays sorted
      SparseOperator& sh = shard_mirror_[owner(spec, all.keys[i], config_.n)];
      sh.keys.push_back(all.keys[i]);
      sh.values.push_back(all.values[i]);
    }
    mirror_valid_ = true;
  }
  return shard_mirror_;
}
std::vector<size_t> Engine::shard_sizes() const {
  std::vector<size_t> out;
  for (const SparseOperator& sh : shards()) out.push_back(sh.term_count());
  return out;
}
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
  out.timers.generate_ns = c.branch_ns;
  out.timers.exchange_ns = c.exchange_ns;
  out.timers.apply_ns = c.other_ns;
  out.timers.truncate_ns = c.truncate_ns;
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
