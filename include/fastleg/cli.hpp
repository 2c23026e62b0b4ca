// Command-line front end of the B200 library, the drop-in for the
// reference's fastleg::cli::run (cli.hpp:111-235): the same subcommands,
// options, defaults, output rows and exit codes
//   0 success, 2 usage error, 3 I/O or file-format error, 4 numerical-domain error
// with an argument parser of its own (the reference's CLI11 dependency is
// not needed). The numerics run on the GPU through the other headers.
#pragma once

#include <algorithm>
#include <array>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "fastleg/fastleg.hpp"

namespace fastleg::cli {

namespace detail {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline std::string shortest(double v) {  // round-trip decimal (std::to_chars)
  std::array<char, 32> buf;
  const auto res = std::to_chars(buf.data(), buf.data() + buf.size(), v);
  return std::string(buf.data(), res.ptr);
}

// Rows of comma-separated fields to a file, or to stdout for "-".
class Rows {
 public:
  explicit Rows(const std::string& target) {
    if (target != "-") {
      file_.open(target);
      if (!file_) throw IoError("cannot open for writing: " + target);
      os_ = &file_;
    }
  }
  void put(const std::vector<std::string>& fields) {
    for (std::size_t i = 0; i < fields.size(); ++i) *os_ << (i ? "," : "") << fields[i];
    *os_ << '\n';
    if (!*os_) throw IoError("write failed");
  }

 private:
  std::ofstream file_;
  std::ostream* os_ = &std::cout;
};

template <class F>
double median_seconds(int reps, F&& body) {
  std::vector<double> t(reps);
  for (double& s : t) {
    const auto a = std::chrono::steady_clock::now();
    body();
    s = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
  }
  std::sort(t.begin(), t.end());
  return t[reps / 2];
}

// One subcommand's options: name -> (value, required, allowed values).
struct Option {
  std::string value;
  bool required = false;
  bool seen = false;
  std::vector<std::string> choices;
  std::string help;
};

struct Command {
  std::string help;
  std::map<std::string, Option> opts;
  std::vector<std::string> order;
  void add(const std::string& name, std::string def, bool required, std::string help,
           std::vector<std::string> choices = {}) {
    opts[name] = Option{std::move(def), required, false, std::move(choices), std::move(help)};
    order.push_back(name);
  }
  const std::string& get(const std::string& name) const { return opts.at(name).value; }
};

inline std::map<std::string, Command> commands() {
  std::map<std::string, Command> c;
  const std::pair<const char*, const char*> transforms[] = {
      {"dlt", "Legendre coefficients -> values at Legendre nodes"},
      {"idlt", "values at Legendre nodes -> Legendre coefficients"},
      {"ndct", "Chebyshev coefficients -> values at Legendre nodes"},
      {"leg2cheb", "Legendre coefficients -> Chebyshev coefficients"}};
  for (const auto& [name, help] : transforms) {
    Command& t = c[name];
    t.help = help;
    t.add("in", "", true, "input vector file");
    t.add("out", "", true, "output vector file");
    t.add("tol", shortest(default_tolerance), false, "working tolerance");
    t.add("grid", "chebstar", false, "reference grid", {"cheb1", "chebstar"});
    t.add("format", "csv", false, "vector file format", {"csv", "bin"});
  }
  Command& nodes = c["nodes"];
  nodes.help = "emit theta, x, w of the N-point Gauss-Legendre rule";
  nodes.add("n", "", true, "number of nodes");
  nodes.add("out", "-", false, "output file ('-' for stdout)");
  Command& cmp = c["compare"];
  cmp.help = "max abs error of the fast transform against the direct evaluation";
  cmp.add("n", "", true, "transform size");
  cmp.add("decay", "1", false, "coefficient decay exponent p, entry n ~ n^-p");
  cmp.add("trials", "5", false, "number of random trials");
  cmp.add("seed", "0", false, "PRNG seed");
  cmp.add("out", "-", false, "output file ('-' for stdout)");
  Command& bench = c["bench"];
  bench.help = "time the fast and direct transforms over a range";
  bench.add("min", "", true, "smallest size");
  bench.add("max", "", true, "largest size");
  bench.add("points", "", true, "number of sizes");
  bench.add("out", "-", false, "output file ('-' for stdout)");
  return c;
}

inline void print_help(std::ostream& os, const std::map<std::string, Command>& cmds,
                       const std::string& sub) {
  if (sub.empty()) {
    os << "fast discrete Legendre transform toolkit (B200)\n"
       << "Usage: fastleg SUBCOMMAND [OPTIONS]\n\nSubcommands:\n";
    for (const auto& [name, cmd] : cmds) os << "  " << name << "  " << cmd.help << '\n';
    return;
  }
  const Command& cmd = cmds.at(sub);
  os << cmd.help << "\nUsage: fastleg " << sub << " [OPTIONS]\n\nOptions:\n";
  for (const std::string& name : cmd.order) {
    const Option& o = cmd.opts.at(name);
    os << "  --" << name << (o.required ? " (required)" : "") << "  " << o.help;
    if (!o.required) os << " [" << o.value << "]";
    os << '\n';
  }
}

template <class T>
T parse_number(const std::string& opt, const std::string& text) {
  T v{};
  const char* end = text.data() + text.size();
  auto res = std::from_chars(text.data(), end, v);
  if (text.empty() || res.ec != std::errc() || res.ptr != end)
    throw UsageError("--" + opt + ": invalid value '" + text + "'");
  return v;
}

inline GridKind grid_of(const std::string& s) {
  return s == "cheb1" ? GridKind::cheb1 : GridKind::chebstar;
}
inline VectorFormat format_of(const std::string& s) {
  return s == "bin" ? VectorFormat::raw_binary : VectorFormat::csv;
}

inline void run_transform(const std::string& name, const Command& cmd) {
  const double tol = parse_number<double>("tol", cmd.get("tol"));
  const GridKind kind = grid_of(cmd.get("grid"));
  const VectorFormat fmt = format_of(cmd.get("format"));
  const std::vector<double> input = read_vector(cmd.get("in"), fmt);
  std::vector<double> output;
  if (name == "leg2cheb") {
    output = leg2cheb_apply(legendre_coefficients(input)).values;
  } else if (name == "ndct") {
    output = ndct_apply(plan_ndct(input.size(), kind, tol), input);
  } else {
    const TransformConfig config(input.size(), tol, kind);
    output = name == "dlt" ? dlt(legendre_coefficients(input), config)
                           : idlt(input, config).values;
  }
  write_vector(cmd.get("out"), output, fmt);
}

}  // namespace detail

inline int run(int argc, const char* const* argv) {
  using namespace detail;
  std::map<std::string, Command> cmds = commands();
  std::string sub;
  // ---- parse (usage errors -> 2, help -> 0)
  try {
    if (argc < 2) throw UsageError("a subcommand is required");
    const std::string first = argv[1];
    if (first == "--help" || first == "-h") {
      print_help(std::cout, cmds, "");
      return 0;
    }
    if (!cmds.count(first)) throw UsageError("unknown subcommand '" + first + "'");
    sub = first;
    Command& cmd = cmds[sub];
    for (int i = 2; i < argc; ++i) {
      std::string a = argv[i];
      if (a == "--help" || a == "-h") {
        print_help(std::cout, cmds, sub);
        return 0;
      }
      if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + a + "'");
      std::string name = a.substr(2), value;
      const std::size_t eq = name.find('=');
      if (eq != std::string::npos) {
        value = name.substr(eq + 1);
        name = name.substr(0, eq);
      } else {
        if (i + 1 >= argc) throw UsageError("--" + name + " needs a value");
        value = argv[++i];
      }
      auto it = cmd.opts.find(name);
      if (it == cmd.opts.end()) throw UsageError("unknown option --" + name + " for " + sub);
      Option& o = it->second;
      if (!o.choices.empty() && std::find(o.choices.begin(), o.choices.end(), value) == o.choices.end())
        throw UsageError("--" + name + ": '" + value + "' is not one of the allowed values");
      o.value = value;
      o.seen = true;
    }
    for (const auto& [name, o] : cmd.opts)
      if (o.required && !o.seen) throw UsageError("--" + name + " is required");
    // numeric options are validated here too (usage, not domain, errors)
    if (sub == "nodes") parse_number<std::size_t>("n", cmd.get("n"));
    if (sub == "compare") {
      parse_number<std::size_t>("n", cmd.get("n"));
      parse_number<double>("decay", cmd.get("decay"));
      parse_number<std::size_t>("trials", cmd.get("trials"));
      parse_number<std::uint64_t>("seed", cmd.get("seed"));
    }
    if (sub == "bench")
      for (const char* k : {"min", "max", "points"}) parse_number<std::size_t>(k, cmd.get(k));
    if (cmd.opts.count("tol")) parse_number<double>("tol", cmd.get("tol"));
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\nRun with --help for more information.\n";
    return 2;
  }

  // ---- run (I/O errors -> 3, everything else -> 4)
  const Command& cmd = cmds.at(sub);
  try {
    if (sub == "dlt" || sub == "idlt" || sub == "ndct" || sub == "leg2cheb") {
      run_transform(sub, cmd);
    } else if (sub == "nodes") {
      const LegendreGrid grid = legendre_nodes_weights(parse_number<std::size_t>("n", cmd.get("n")));
      Rows rows(cmd.get("out"));
      for (std::size_t k = 0; k < grid.size; ++k)
        rows.put({shortest(grid.theta[k]), shortest(grid.x[k]), shortest(grid.weights[k])});
    } else if (sub == "compare") {
      const std::size_t n = parse_number<std::size_t>("n", cmd.get("n"));
      const double decay = parse_number<double>("decay", cmd.get("decay"));
      const std::size_t trials = parse_number<std::size_t>("trials", cmd.get("trials"));
      GaussianSource source(parse_number<std::uint64_t>("seed", cmd.get("seed")));
      const TransformConfig config(n);
      Rows rows(cmd.get("out"));
      for (std::size_t t = 0; t < trials; ++t) {
        const CoefficientVector c = legendre_coefficients(random_decaying(n, decay, source));
        const std::vector<double> fast = dlt(c, config);
        const std::vector<double> direct = eval_legendre_direct(c, config.grid().x);
        double err = 0.0;
        for (std::size_t k = 0; k < fast.size(); ++k) err = std::max(err, std::fabs(fast[k] - direct[k]));
        rows.put({std::to_string(n), shortest(err)});
      }
    } else {  // bench
      const std::size_t lo = parse_number<std::size_t>("min", cmd.get("min"));
      const std::size_t hi = parse_number<std::size_t>("max", cmd.get("max"));
      const std::size_t points = parse_number<std::size_t>("points", cmd.get("points"));
      if (lo == 0 || hi < lo || points == 0)
        throw std::invalid_argument("bench: need 0 < min <= max and points >= 1");
      std::vector<std::size_t> sizes;  // log-spaced, rounded, deduplicated
      for (std::size_t i = 0; i < points; ++i) {
        const double f = points == 1 ? 0.0 : (double)i / (double)(points - 1);
        const double l = std::log((double)lo) + f * (std::log((double)hi) - std::log((double)lo));
        const auto n = (std::size_t)std::llround(std::exp(l));
        if (sizes.empty() || sizes.back() != n) sizes.push_back(n);
      }
      Rows rows(cmd.get("out"));
      for (std::size_t n : sizes) {
        const TransformConfig config(n);
        const CoefficientVector c = legendre_coefficients(random_decaying(n, 1.0, 7));
        std::vector<double> sink;
        const double fast = median_seconds(5, [&] { sink = dlt(c, config); });
        const double direct =
            median_seconds(5, [&] { sink = eval_legendre_direct(c, config.grid().x); });
        rows.put({std::to_string(n), shortest(fast), shortest(direct)});
      }
    }
  } catch (const IoError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 4;
  }
  return 0;
}

}  // namespace fastleg::cli
