// lvn_cli: the reference's command line front end (tools/louvain_cli.cpp)
// over the B200 engine, through the C-ABI of include/lvn.h only.
//
//   lvn_cli detect  --input G [--format mtx|tsv] [--engine gpu] [params] [--output M.tsv] [--report R]
//   lvn_cli bench   --input G [params] [--threads 1,2] [--repetitions 5] [--report R]
//   lvn_cli convert --input G --output H [--symmetrize]
//
// Same report schema (flat key=value lines; bench adds row=run / row=scaling
// lines), same loaders (io.cpp:54-137: MatrixMarket coordinate real|integer|
// pattern, general|symmetric, 1-based; whitespace TSV "src dst [weight]",
// 0-based, '#' comments), same exit codes (louvain_cli.cpp:343-355):
// 0 ok, 1 parse / invalid argument, 2 degenerate graph, 3 internal invariant.
// CUDA failures exit 4. The graph is built on the device (lvn_build_csr,
// build_csr of graph.cpp:15-87) and symmetrized like the reference's detect.
// --engine accepts gpu (the default); --threads is echoed in the report for
// schema parity (the device engine has no host worker team).
#include <algorithm>
#include <cctype>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "lvn.h"

namespace {

constexpr int kExitParse = 1, kExitDegenerate = 2, kExitInternal = 3, kExitCuda = 4;

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct LvnError : std::runtime_error {
  int code;
  LvnError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(int rc) {
  if (rc != LVN_OK) throw LvnError(rc, lvn_last_error());
}

std::string at_line(const std::string& what, std::size_t line) {
  return line ? what + " (line " + std::to_string(line) + ")" : what;
}

// ---- edge lists (io.cpp) ------------------------------------------------------
struct EdgeList {
  std::uint32_t n = 0;
  std::vector<std::uint32_t> src, dst;
  std::vector<double> w;
};

std::string lower(std::string_view s) {
  std::string out(s);
  for (auto& c : out) c = char(std::tolower(static_cast<unsigned char>(c)));
  return out;
}

std::vector<std::string_view> split_ws(std::string_view line) {
  std::vector<std::string_view> t;
  std::size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
    std::size_t j = i;
    while (j < line.size() && !std::isspace(static_cast<unsigned char>(line[j]))) ++j;
    if (j > i) t.push_back(line.substr(i, j - i));
    i = j;
  }
  return t;
}

std::uint64_t parse_uint(std::string_view tok, std::size_t line) {
  std::uint64_t v = 0;
  auto [p, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (ec != std::errc{} || p != tok.data() + tok.size())
    throw ParseError(at_line("expected an unsigned integer, got '" + std::string(tok) + "'", line));
  return v;
}

double parse_weight(std::string_view tok, std::size_t line) {
  double v = 0.0;
  auto [p, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (ec != std::errc{} || p != tok.data() + tok.size())
    throw ParseError(at_line("expected a number, got '" + std::string(tok) + "'", line));
  if (v < 0.0) throw ParseError(at_line("negative edge weight", line));
  return v;
}

constexpr std::uint64_t kInvalidVertex = 0xFFFFFFFFull;

EdgeList load_mtx(std::istream& in) {
  std::string line;
  std::size_t ln = 0;
  if (!std::getline(in, line)) throw ParseError(at_line("empty file", 1));
  ++ln;
  auto banner = split_ws(line);
  if (banner.size() < 4 || lower(banner[0]) != "%%matrixmarket" || lower(banner[1]) != "matrix")
    throw ParseError(at_line("missing %%MatrixMarket matrix banner", ln));
  if (lower(banner[2]) != "coordinate") throw ParseError(at_line("only coordinate format is supported", ln));
  const std::string field = lower(banner[3]);
  if (field != "real" && field != "integer" && field != "pattern")
    throw ParseError(at_line("unsupported field '" + field + "'", ln));
  const std::string sym = banner.size() > 4 ? lower(banner[4]) : "general";
  if (sym != "general" && sym != "symmetric") throw ParseError(at_line("unsupported symmetry '" + sym + "'", ln));
  std::uint64_t rows = 0, cols = 0, entries = 0;
  for (;;) {
    if (!std::getline(in, line)) throw ParseError(at_line("missing size line", ln));
    ++ln;
    if (!line.empty() && line[0] == '%') continue;
    auto t = split_ws(line);
    if (t.empty()) continue;
    if (t.size() != 3) throw ParseError(at_line("size line must be 'rows cols entries'", ln));
    rows = parse_uint(t[0], ln), cols = parse_uint(t[1], ln), entries = parse_uint(t[2], ln);
    break;
  }
  if (rows != cols) throw ParseError(at_line("adjacency matrix must be square", ln));
  if (rows >= kInvalidVertex) throw ParseError(at_line("vertex count out of range", ln));
  EdgeList el;
  el.n = std::uint32_t(rows);
  el.src.reserve(entries), el.dst.reserve(entries), el.w.reserve(entries);
  const bool want_weight = field != "pattern";
  std::uint64_t seen = 0;
  while (seen < entries) {
    if (!std::getline(in, line)) throw ParseError(at_line("unexpected end of file", ln));
    ++ln;
    if (!line.empty() && line[0] == '%') continue;
    auto t = split_ws(line);
    if (t.empty()) continue;
    if (t.size() < 2 || t.size() > 3 || (!want_weight && t.size() != 2))
      throw ParseError(at_line(std::string("entry must be 'row col") + (want_weight ? " [value]'" : "'"), ln));
    const std::uint64_t r = parse_uint(t[0], ln), c = parse_uint(t[1], ln);
    if (r < 1 || r > rows || c < 1 || c > cols) throw ParseError(at_line("entry id out of declared bounds", ln));
    el.src.push_back(std::uint32_t(r - 1));
    el.dst.push_back(std::uint32_t(c - 1));
    el.w.push_back(t.size() == 3 ? parse_weight(t[2], ln) : 1.0);
    ++seen;
  }
  return el;
}

EdgeList load_tsv(std::istream& in) {
  EdgeList el;
  std::string line;
  std::size_t ln = 0;
  std::uint64_t max_id = 0;
  bool any = false;
  while (std::getline(in, line)) {
    ++ln;
    auto t = split_ws(line);
    if (t.empty() || t[0].front() == '#') continue;
    if (t.size() < 2 || t.size() > 3) throw ParseError(at_line("line must be 'src dst [weight]'", ln));
    const std::uint64_t u = parse_uint(t[0], ln), v = parse_uint(t[1], ln);
    if (u >= kInvalidVertex || v >= kInvalidVertex) throw ParseError(at_line("vertex id out of range", ln));
    el.src.push_back(std::uint32_t(u));
    el.dst.push_back(std::uint32_t(v));
    el.w.push_back(t.size() == 3 ? parse_weight(t[2], ln) : 1.0);
    max_id = std::max({max_id, u, v});
    any = true;
  }
  el.n = any ? std::uint32_t(max_id + 1) : 0;
  return el;
}

bool is_mtx(const std::string& path) {
  const auto dot = path.rfind('.');
  return dot != std::string::npos && lower(path.substr(dot)) == ".mtx";
}

EdgeList load_edge_list(const std::string& path, const std::string& format) {
  bool mtx = is_mtx(path);
  if (format == "mtx") mtx = true;
  else if (format == "tsv") mtx = false;
  else if (!format.empty()) throw ParseError("unknown format '" + format + "' (expected mtx or tsv)");
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open '" + path + "'");
  return mtx ? load_mtx(in) : load_tsv(in);
}

void write_weight(std::string& out, double w) {
  char buf[32];
  auto [p, ec] = std::to_chars(buf, buf + sizeof buf, w);  // shortest round-trip form
  out.append(buf, p);
}

void save_edges(const std::string& path, const EdgeList& e) {
  std::ofstream out(path);
  if (!out) throw ParseError("cannot write '" + path + "'");
  std::string body;
  if (is_mtx(path)) {
    body = "%%MatrixMarket matrix coordinate real general\n" + std::to_string(e.n) + " " + std::to_string(e.n) +
           " " + std::to_string(e.src.size()) + "\n";
    for (std::size_t i = 0; i < e.src.size(); ++i) {
      body += std::to_string(e.src[i] + 1ull) + " " + std::to_string(e.dst[i] + 1ull) + " ";
      write_weight(body, e.w[i]);
      body += '\n';
    }
  } else {
    body = "# vertices: " + std::to_string(e.n) + "\n";
    for (std::size_t i = 0; i < e.src.size(); ++i) {
      body += std::to_string(e.src[i]) + "\t" + std::to_string(e.dst[i]) + "\t";
      write_weight(body, e.w[i]);
      body += '\n';
    }
  }
  out << body;
  if (!out) throw ParseError("write failed for '" + path + "'");
}

// ---- CSR on the host (library-owned arrays from lvn_build_csr) -------------------
struct Graph {
  lvn_graph_out* g = nullptr;
  ~Graph() { lvn_graph_free(g); }
  lvn_csr view() const {
    lvn_csr v{};
    v.num_vertices = g->num_vertices;
    v.num_arcs = g->num_arcs;
    v.offsets = g->offsets;
    v.targets = g->targets;
    v.weights = g->weights;
    v.total_weight = g->total_weight;
    v.location = LVN_HOST;
    return v;
  }
};

void build(const EdgeList& e, bool symmetrize, Graph& out) {
  check(lvn_build_csr(e.n, e.src.size(), e.src.data(), e.dst.data(), e.w.data(), symmetrize ? 1 : 0, &out.g));
}

// ---- options ------------------------------------------------------------------
struct Options {
  std::string cmd, input, format, engine = "gpu", threads, output, report, probing = "quadratic-double";
  int max_passes = 10, max_iterations = 20, pl_period = 4, value_bits = 32, repetitions = 5, gpus = 1;
  double tolerance = 0.01, tolerance_drop = 10.0, aggregation_tolerance = 0.8;
  std::uint64_t switch_move = 64, switch_aggregate = 128;
  bool symmetrize = false;
};

int probing_code(const std::string& p) {
  if (p == "linear") return 0;
  if (p == "quadratic") return 1;
  if (p == "double") return 2;
  if (p == "quadratic-double") return 3;
  throw ParseError("unknown probing mode '" + p + "'");
}

std::vector<int> thread_list(const std::string& list) {
  if (list.empty()) return {0};
  std::vector<int> out;
  std::stringstream in(list);
  std::string tok;
  while (std::getline(in, tok, ',')) {
    std::size_t used = 0;
    int v = 0;
    try {
      v = std::stoi(tok, &used);
    } catch (const std::exception&) {
      throw ParseError("bad thread count '" + tok + "'");
    }
    if (used != tok.size() || v < 0) throw ParseError("bad thread count '" + tok + "'");
    out.push_back(v);
  }
  if (out.empty()) throw ParseError("empty thread list");
  return out;
}

Options parse_args(int argc, char** argv) {
  if (argc < 2) throw ParseError("usage: lvn_cli detect|bench|convert --input PATH [options]");
  Options o;
  o.cmd = argv[1];
  if (o.cmd != "detect" && o.cmd != "bench" && o.cmd != "convert") throw ParseError("unknown subcommand '" + o.cmd + "'");
  if (const char* e = std::getenv("LOUVAIN_THREADS")) o.threads = e;
  auto need = [&](int& i) -> std::string {
    if (i + 1 >= argc) throw ParseError(std::string(argv[i]) + " needs a value");
    return argv[++i];
  };
  auto num = [](const std::string& flag, const std::string& v, auto& dst) {
    std::istringstream in(v);
    in >> dst;
    if (!in || !in.eof()) throw ParseError("bad value '" + v + "' for " + flag);
  };
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--input") o.input = need(i);
    else if (a == "--format") o.format = need(i);
    else if (a == "--engine") o.engine = need(i);
    else if (a == "--threads") o.threads = need(i);
    else if (a == "--gpus") num(a, need(i), o.gpus);
    else if (a == "--max-passes") num(a, need(i), o.max_passes);
    else if (a == "--max-iterations") num(a, need(i), o.max_iterations);
    else if (a == "--tolerance") num(a, need(i), o.tolerance);
    else if (a == "--tolerance-drop") num(a, need(i), o.tolerance_drop);
    else if (a == "--aggregation-tolerance") num(a, need(i), o.aggregation_tolerance);
    else if (a == "--pl-period") num(a, need(i), o.pl_period);
    else if (a == "--switch-move") num(a, need(i), o.switch_move);
    else if (a == "--switch-aggregate") num(a, need(i), o.switch_aggregate);
    else if (a == "--probing") o.probing = need(i);
    else if (a == "--value-bits") num(a, need(i), o.value_bits);
    else if (a == "--output") o.output = need(i);
    else if (a == "--report") o.report = need(i);
    else if (a == "--repetitions") num(a, need(i), o.repetitions);
    else if (a == "--symmetrize") o.symmetrize = true;
    else throw ParseError("unknown option '" + a + "'");
  }
  if (o.input.empty()) throw ParseError("--input is required");
  if (o.engine != "gpu") throw ParseError("unknown engine '" + o.engine + "' (this build runs the gpu engine)");
  if (o.gpus != 1)
    throw ParseError("--gpus: one device per process; run several processes with lvn_louvain_sharded for more");
  probing_code(o.probing);
  return o;
}

lvn_params params_of(const Options& o, int threads) {
  lvn_params p;
  lvn_params_default(&p);
  p.max_passes = o.max_passes;
  p.max_iterations = o.max_iterations;
  p.initial_tolerance = o.tolerance;
  p.tolerance_drop = o.tolerance_drop;
  p.aggregation_tolerance = o.aggregation_tolerance;
  p.thread_count = threads;
  p.pick_less_period = o.pl_period;
  p.switch_move = o.switch_move;
  p.switch_aggregate = o.switch_aggregate;
  p.probing = probing_code(o.probing);
  p.value_bits = o.value_bits;
  return p;
}

// ---- report (louvain_cli.cpp:139-177) -------------------------------------------
template <class T>
std::string join(const T* v, std::size_t n) {
  std::ostringstream out;
  out.precision(12);
  for (std::size_t i = 0; i < n; ++i) out << (i ? "," : "") << v[i];
  return out.str();
}

void describe_input(std::ostream& out, const Options& o, const lvn_graph_out* g) {
  out << "input=" << o.input << "\n";
  out << "vertices=" << g->num_vertices << "\n";
  out << "edges=" << double(g->num_arcs) / 2.0 << "\n";
  out << "avg_degree=" << (g->num_vertices ? double(g->num_arcs) / g->num_vertices : 0.0) << "\n";
  out << "engine=" << o.engine << "\n";
}

void describe_params(std::ostream& out, const Options& o, int threads) {
  out << "threads=" << threads << "\n";
  out << "gpus=" << o.gpus << "\n";
  out << "max_passes=" << o.max_passes << "\n";
  out << "max_iterations=" << o.max_iterations << "\n";
  out << "tolerance=" << o.tolerance << "\n";
  out << "tolerance_drop=" << o.tolerance_drop << "\n";
  out << "aggregation_tolerance=" << o.aggregation_tolerance << "\n";
  out << "pl_period=" << o.pl_period << "\n";
  out << "switch_move=" << o.switch_move << "\n";
  out << "switch_aggregate=" << o.switch_aggregate << "\n";
  out << "probing=" << o.probing << "\n";
  out << "value_bits=" << o.value_bits << "\n";
}

void describe_result(std::ostream& out, const lvn_graph_out* g, const lvn_result* r) {
  const double wall = r->wall_seconds > 0 ? r->wall_seconds : 1e-300;
  out << "modularity=" << r->modularity << "\n";
  out << "communities=" << r->num_communities << "\n";
  out << "passes=" << r->passes << "\n";
  out << "iterations_per_pass=" << join(r->iterations_per_pass, std::size_t(r->passes)) << "\n";
  out << "phase_local_moving=" << r->local_moving / wall << "\n";
  out << "phase_aggregation=" << r->aggregation / wall << "\n";
  out << "phase_other=" << r->other / wall << "\n";
  std::vector<double> split(std::size_t(r->passes));
  for (std::size_t i = 0; i < split.size(); ++i) split[i] = r->pass_seconds[i] / wall;
  out << "pass_split=" << join(split.data(), split.size()) << "\n";
  out << "wall_time=" << r->wall_seconds << "\n";
  out << "edges_per_second=" << (double(g->num_arcs) / 2.0) / wall << "\n";
}

// the emitted membership is a contiguous renumbering whose recomputed
// modularity matches the reported value (louvain_cli.cpp:179-196)
void verify(const Graph& g, const lvn_result* r) {
  if (r->num_vertices != g.g->num_vertices) throw LvnError(LVN_INTERNAL, "membership size does not match the graph");
  std::vector<char> seen(r->num_communities, 0);
  for (std::uint32_t v = 0; v < r->num_vertices; ++v) {
    const std::uint32_t c = r->membership[v];
    if (c >= r->num_communities) throw LvnError(LVN_INTERNAL, "membership is not a contiguous renumbering");
    seen[c] = 1;
  }
  if (!std::all_of(seen.begin(), seen.end(), [](char b) { return b != 0; }))
    throw LvnError(LVN_INTERNAL, "membership is not a contiguous renumbering");
  const lvn_csr v = g.view();
  double q = 0.0;
  check(lvn_modularity(&v, r->membership, LVN_HOST, &q));
  if (std::abs(q - r->modularity) > 1e-9) throw LvnError(LVN_INTERNAL, "reported modularity diverges from the membership file");
}

void save_membership(const std::string& path, const lvn_result* r) {
  std::ofstream out(path);
  if (!out) throw ParseError("cannot write '" + path + "'");
  std::string body;
  for (std::uint32_t v = 0; v < r->num_vertices; ++v)
    body += std::to_string(v) + "\t" + std::to_string(r->membership[v]) + "\n";
  out << body;
  if (!out) throw ParseError("write failed for '" + path + "'");
}

void emit(const std::string& path, const std::string& text) {
  if (path.empty()) {
    std::cout << text;
    return;
  }
  std::ofstream out(path);
  if (!out) throw ParseError("cannot open report path " + path);
  out << text;
}

struct Result {
  lvn_result* r = nullptr;
  ~Result() { lvn_result_free(r); }
};

int cmd_detect(const Options& o) {
  const EdgeList e = load_edge_list(o.input, o.format);
  Graph g;
  build(e, true, g);
  const auto threads = thread_list(o.threads);
  if (threads.size() != 1) throw ParseError("detect takes a single --threads value");
  const lvn_params p = params_of(o, threads.front());
  const lvn_csr v = g.view();
  Result r;
  check(lvn_louvain(&v, &p, &r.r));
  verify(g, r.r);
  if (!o.output.empty()) save_membership(o.output, r.r);
  std::ostringstream rep;
  rep.precision(12);
  describe_input(rep, o, g.g);
  describe_params(rep, o, threads.front());
  describe_result(rep, g.g, r.r);
  emit(o.report, rep.str());
  return 0;
}

int cmd_bench(const Options& o) {
  const EdgeList e = load_edge_list(o.input, o.format);
  Graph g;
  build(e, true, g);
  const auto threads = thread_list(o.threads);
  if (o.repetitions < 1) throw ParseError("--repetitions must be at least 1");
  std::ostringstream rep;
  rep.precision(12);
  describe_input(rep, o, g.g);
  describe_params(rep, o, threads.front());
  rep << "repetitions=" << o.repetitions << "\n";
  struct Agg {
    double geo = 0, q = 0, lm = 0, ag = 0, ot = 0;
  };
  std::vector<std::pair<int, Agg>> table;
  const lvn_csr v = g.view();
  for (const int t : threads) {
    const lvn_params p = params_of(o, t);
    Agg a;
    double logw = 0;
    for (int k = 0; k < o.repetitions; ++k) {
      Result r;
      check(lvn_louvain(&v, &p, &r.r));
      verify(g, r.r);
      const double wall = r.r->wall_seconds > 0 ? r.r->wall_seconds : 1e-300;
      rep << "row=run threads=" << t << " rep=" << k + 1 << " wall_time=" << r.r->wall_seconds
          << " modularity=" << r.r->modularity << " passes=" << r.r->passes << "\n";
      logw += std::log(wall);
      a.q += r.r->modularity;
      a.lm += r.r->local_moving / wall;
      a.ag += r.r->aggregation / wall;
      a.ot += r.r->other / wall;
    }
    a.geo = std::exp(logw / o.repetitions);
    a.q /= o.repetitions, a.lm /= o.repetitions, a.ag /= o.repetitions, a.ot /= o.repetitions;
    table.emplace_back(t, a);
  }
  auto ref = std::find_if(table.begin(), table.end(), [](const auto& r) { return r.first == 1; });
  const double base = (ref != table.end() ? ref : table.begin())->second.geo;
  for (const auto& [t, a] : table)
    rep << "row=scaling threads=" << t << " runs=" << o.repetitions << " wall_time_geomean=" << a.geo
        << " modularity_mean=" << a.q << " phase_local_moving=" << a.lm << " phase_aggregation=" << a.ag
        << " phase_other=" << a.ot << " speedup=" << base / a.geo << "\n";
  emit(o.report, rep.str());
  return 0;
}

int cmd_convert(const Options& o) {
  if (o.output.empty()) throw ParseError("convert requires --output");
  EdgeList e = load_edge_list(o.input, o.format);
  if (o.symmetrize) {  // to_edge_list(build_csr(edges, true)): one triple per arc
    Graph g;
    build(e, true, g);
    EdgeList s;
    s.n = g.g->num_vertices;
    for (std::uint32_t u = 0; u < s.n; ++u)
      for (std::uint64_t a = g.g->offsets[u]; a < g.g->offsets[u + 1]; ++a) {
        s.src.push_back(u);
        s.dst.push_back(g.g->targets[a]);
        s.w.push_back(double(g.g->weights[a]));
      }
    e = std::move(s);
  }
  save_edges(o.output, e);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Options o = parse_args(argc, argv);
    if (o.cmd == "detect") return cmd_detect(o);
    if (o.cmd == "bench") return cmd_bench(o);
    return cmd_convert(o);
  } catch (const ParseError& e) {
    std::cerr << "parse error: " << e.what() << "\n";
    return kExitParse;
  } catch (const LvnError& e) {
    switch (e.code) {
      case LVN_INVALID_ARGUMENT: std::cerr << "parse error: " << e.what() << "\n"; return kExitParse;
      case LVN_DEGENERATE: std::cerr << "degenerate graph: " << e.what() << "\n"; return kExitDegenerate;
      case LVN_INTERNAL: std::cerr << "internal error: " << e.what() << "\n"; return kExitInternal;
      default: std::cerr << "cuda error: " << e.what() << "\n"; return kExitCuda;
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitParse;
  }
}
