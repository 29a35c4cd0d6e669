// anisoq_b200: the reference command-line tool's hot-path verbs on the B200
// (reference proj/tools/anisoq_main.cpp). Same verbs, option names, defaults,
// output files and exit codes (0 ok, 2 validation error, 3 runtime error):
//
//   gen     synthetic fvecs (anisoq_main.cpp:232-261)
//   train   train_apq / train_avq -> codebook.bin, codes.bin, train_log.csv,
//           manifest.json (358-425)
//   encode  pq_quantize -> codes + <out>.meta.json (427-454)
//   search  adc_search per query, one line per hit (456-478)
//   eval    exact ground truth (cached as ivecs) + evaluate -> eval_report.txt,
//           eval_report.json, manifest.json (480-579)
//
// Every data-parallel step runs through libanisoq_b200.so (the C++ drop-in
// headers under include/anisoq); search issues all queries as one device
// batch (bit-identical to the per-query loop). The reference's convert,
// diagnose and eta verbs are outside the hot path and are
// rejected with a validation error. `--config` reads the reference's JSON
// documents (a section per verb, or top-level keys; explicit flags win).
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "anisoq/anisoq.hpp"

namespace fs = std::filesystem;

namespace {

constexpr int kExitValidation = 2;
constexpr int kExitRuntime = 3;

// ---- minimal JSON value (config documents in, manifests out) ------------------------

struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  std::string raw;  // number text as written (integers stay exact)
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  const Json* find(const std::string& k) const {
    for (const auto& [key, v] : obj)
      if (key == k) return &v;
    return nullptr;
  }
};

struct JsonParser {
  const std::string& s;
  size_t i = 0;
  std::string where;

  [[noreturn]] void fail(const std::string& m) {
    throw anisoq::MalformedFile("config " + where + ": " + m + " at offset " + std::to_string(i));
  }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  Json value() {
    ws();
    if (i >= s.size()) fail("unexpected end");
    const char c = s[i];
    Json v;
    if (c == '{') {
      v.kind = Json::Obj;
      ++i;
      ws();
      if (i < s.size() && s[i] == '}') {
        ++i;
        return v;
      }
      for (;;) {
        ws();
        if (i >= s.size() || s[i] != '"') fail("expected key");
        std::string k = string();
        ws();
        if (i >= s.size() || s[i] != ':') fail("expected ':'");
        ++i;
        v.obj.emplace_back(k, value());
        ws();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == '}') {
          ++i;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Json::Arr;
      ++i;
      ws();
      if (i < s.size() && s[i] == ']') {
        ++i;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == ']') {
          ++i;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Json::Str;
      v.str = string();
      return v;
    }
    if (s.compare(i, 4, "true") == 0) {
      i += 4;
      v.kind = Json::Bool;
      v.b = true;
      return v;
    }
    if (s.compare(i, 5, "false") == 0) {
      i += 5;
      v.kind = Json::Bool;
      return v;
    }
    if (s.compare(i, 4, "null") == 0) {
      i += 4;
      return v;
    }
    const size_t b = i;
    while (i < s.size() && (std::isdigit(static_cast<unsigned char>(s[i])) || s[i] == '-' ||
                            s[i] == '+' || s[i] == '.' || s[i] == 'e' || s[i] == 'E'))
      ++i;
    if (b == i) fail("unexpected character");
    v.kind = Json::Num;
    v.raw = s.substr(b, i - b);
    char* end = nullptr;
    v.num = std::strtod(v.raw.c_str(), &end);
    if (end != v.raw.c_str() + v.raw.size()) fail("bad number");
    return v;
  }
  std::string string() {
    ++i;  // opening quote
    std::string out;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\') {
        if (++i >= s.size()) break;
        const char e = s[i];
        out += e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e;
      } else {
        out += s[i];
      }
      ++i;
    }
    if (i >= s.size()) fail("unterminated string");
    ++i;
    return out;
  }
};

// Output side: a document written like nlohmann::json::dump(2) (keys in
// sorted order, as the reference's std::map-backed json objects print).
struct Doc {
  std::vector<std::pair<std::string, std::string>> items;  // key -> serialized value
  Doc& add(const std::string& k, const std::string& serialized) {
    items.emplace_back(k, serialized);
    std::stable_sort(items.begin(), items.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    return *this;
  }
  std::string dump(int indent = 2, int level = 0) const {
    if (items.empty()) return "{}";
    const std::string pad((level + 1) * indent, ' '), end(level * indent, ' ');
    std::string out = "{\n";
    for (size_t t = 0; t < items.size(); ++t) {
      out += pad + quote(items[t].first) + ": " + reindent(items[t].second, pad);
      out += t + 1 < items.size() ? ",\n" : "\n";
    }
    return out + end + "}";
  }
  static std::string quote(const std::string& v) {
    std::string o = "\"";
    for (char c : v) {
      if (c == '"' || c == '\\') o += '\\';
      if (c == '\n') {
        o += "\\n";
        continue;
      }
      o += c;
    }
    return o + "\"";
  }
  static std::string reindent(const std::string& v, const std::string& pad) {
    std::string o;
    for (char c : v) {
      o += c;
      if (c == '\n') o += pad;
    }
    return o;
  }
};

// shortest representation that reads back to the same double (nlohmann's dump)
std::string jnum(double v) {
  char buf[40];
  for (int p = 1; p <= 17; ++p) {
    std::snprintf(buf, sizeof buf, "%.*g", p, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}
std::string jint(long long v) { return std::to_string(v); }
std::string jbool(bool v) { return v ? "true" : "false"; }
std::string jstr(const std::string& v) { return Doc::quote(v); }
std::string jarr(const std::vector<std::string>& v) {
  std::string o = "[\n";
  for (size_t t = 0; t < v.size(); ++t) o += "  " + v[t] + (t + 1 < v.size() ? ",\n" : "\n");
  return o + "]";
}

std::string file_digest(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw anisoq::MalformedFile("cannot open " + path);
  std::vector<char> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  std::uint64_t h = 0xcbf29ce484222325ull;  // fnv1a64 (reference dataset.hpp:62-70)
  for (char c : bytes) {
    h ^= static_cast<unsigned char>(c);
    h *= 0x100000001b3ull;
  }
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(h));
  return buf;
}

void write_json(const Doc& doc, const std::string& path) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw anisoq::MalformedFile("cannot open " + path + " for writing");
  out << doc.dump() << "\n";
}

// ---- options -------------------------------------------------------------------------

struct Opt {
  std::string name;  // long name without dashes (also the config key)
  bool flag = false;
  bool required = false;
  bool seen = false;
  bool negatable = false;  // --x / --no-x
  std::function<void(const std::string&)> set;
  std::function<void(const Json&)> from_json;
};

template <class T>
T parse_as(const std::string& name, const std::string& v);
template <>
double parse_as(const std::string& name, const std::string& v) {
  char* e = nullptr;
  const double r = std::strtod(v.c_str(), &e);
  if (v.empty() || *e) throw anisoq::InvalidArgument("--" + name + ": not a number: " + v);
  return r;
}
template <>
long parse_as(const std::string& name, const std::string& v) {
  char* e = nullptr;
  const long r = std::strtol(v.c_str(), &e, 10);
  if (v.empty() || *e) throw anisoq::InvalidArgument("--" + name + ": not an integer: " + v);
  return r;
}

struct Verb {
  std::string name;
  std::vector<Opt> opts;
  std::string config;

  template <class T>
  void opt(const std::string& n, T& target, bool required = false) {
    Opt o;
    o.name = n;
    o.required = required;
    o.set = [&target, n](const std::string& v) {
      if constexpr (std::is_same_v<T, std::string>) {
        target = v;
      } else if constexpr (std::is_floating_point_v<T>) {
        target = static_cast<T>(parse_as<double>(n, v));
      } else {
        const long r = parse_as<long>(n, v);
        if (std::is_unsigned_v<T> && r < 0)
          throw anisoq::InvalidArgument("--" + n + ": must be >= 0");
        target = static_cast<T>(r);
      }
    };
    o.from_json = [&target, n](const Json& j) {
      if constexpr (std::is_same_v<T, std::string>) {
        if (j.kind != Json::Str) throw anisoq::MalformedFile("config key " + n + ": expected a string");
        target = j.str;
      } else {
        if (j.kind != Json::Num) throw anisoq::MalformedFile("config key " + n + ": expected a number");
        if constexpr (std::is_floating_point_v<T>) {
          target = static_cast<T>(j.num);
        } else {
          if (j.num < 0 && std::is_unsigned_v<T>)
            throw anisoq::MalformedFile("config key " + n + ": must be >= 0");
          target = static_cast<T>(std::strtoll(j.raw.c_str(), nullptr, 10));
        }
      }
    };
    opts.push_back(std::move(o));
  }
  void flag(const std::string& n, bool& target, bool negatable = false) {
    Opt o;
    o.name = n;
    o.flag = true;
    o.negatable = negatable;
    o.set = [&target](const std::string& v) { target = v != "false"; };
    o.from_json = [&target, n](const Json& j) {
      if (j.kind != Json::Bool) throw anisoq::MalformedFile("config key " + n + ": expected a bool");
      target = j.b;
    };
    opts.push_back(std::move(o));
  }

  void parse(int argc, char** argv, int first) {
    for (int a = first; a < argc; ++a) {
      std::string t = argv[a];
      if (t.rfind("--", 0) != 0) throw anisoq::InvalidArgument("unexpected argument " + t);
      std::string key = t.substr(2), val;
      const size_t eq = key.find('=');
      bool has_val = eq != std::string::npos;
      if (has_val) {
        val = key.substr(eq + 1);
        key = key.substr(0, eq);
      }
      if (key == "config") {
        if (!has_val) {
          if (a + 1 >= argc) throw anisoq::InvalidArgument("--config needs a value");
          val = argv[++a];
        }
        config = val;
        continue;
      }
      if (key == "T" || key == "help") throw anisoq::InvalidArgument("unknown option --" + key);
      Opt* o = nullptr;
      bool negate = false;
      for (auto& c : opts) {
        if (c.name == key) o = &c;
        if (c.negatable && "no-" + c.name == key) {
          o = &c;
          negate = true;
        }
      }
      if (!o) throw anisoq::InvalidArgument("unknown option --" + key + " for " + name);
      if (o->flag) {
        o->set(negate ? "false" : (has_val ? val : "true"));
      } else {
        if (!has_val) {
          if (a + 1 >= argc) throw anisoq::InvalidArgument("--" + key + " needs a value");
          val = argv[++a];
        }
        o->set(val);
      }
      o->seen = true;
    }
  }

  // apply_config (anisoq_main.cpp:75-98): section values, then top-level
  // scalars, for options not given on the command line.
  void apply_config() {
    if (config.empty()) return;
    std::ifstream in(config);
    if (!in) throw anisoq::MalformedFile("cannot open config " + config);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    JsonParser p{text, 0, config};
    const Json root = p.value();
    if (root.kind != Json::Obj) throw anisoq::MalformedFile("config " + config + ": not an object");
    const Json* sub = root.find(name);
    if (sub && sub->kind != Json::Obj) sub = nullptr;
    for (auto& o : opts) {
      if (o.seen) continue;
      const Json* v = sub ? sub->find(o.name) : nullptr;
      if (!v) {
        v = root.find(o.name);
        if (v && v->kind == Json::Obj) v = nullptr;
      }
      if (v) {
        o.from_json(*v);
        o.seen = true;
      }
    }
    for (const auto& o : opts)
      if (o.required && !o.seen) throw anisoq::InvalidArgument("--" + o.name + " is required");
  }

  void check_required() const {
    if (!config.empty()) return;  // checked after the config is applied
    for (const auto& o : opts)
      if (o.required && !o.seen) throw anisoq::InvalidArgument("--" + o.name + " is required");
  }
};

// ---- verbs ---------------------------------------------------------------------------

struct LossSpec {
  std::string loss = "score_aware";  // or "reconstruction"
  double threshold = 0.2;
  double explicit_eta = -1.0;
};

// resolve_weights (anisoq_main.cpp:108-142): h_perp = 1, h_par = eta.
std::vector<anisoq::AnisotropicWeights> resolve_weights(const LossSpec& spec,
                                                        const anisoq::Dataset& data, Doc* meta) {
  using anisoq::AnisotropicWeights;
  std::vector<AnisotropicWeights> w;
  w.reserve(data.n);
  if (spec.loss == "reconstruction") {
    w.assign(data.n, AnisotropicWeights::isotropic());
    if (meta) meta->add("loss", jstr("reconstruction"));
    return w;
  }
  if (spec.loss != "score_aware")
    throw anisoq::InvalidArgument("loss must be reconstruction or score_aware");
  if (meta) meta->add("loss", jstr("score_aware"));
  if (spec.explicit_eta >= 0.0) {
    w.assign(data.n, AnisotropicWeights::from_eta(spec.explicit_eta));
    if (meta) meta->add("eta", jnum(spec.explicit_eta));
    return w;
  }
  double lo = 0.0, hi = 0.0, sum = 0.0;
  for (std::size_t i = 0; i < data.n; ++i) {
    const double eta = anisoq::eta_limit(spec.threshold, data.norms[i], static_cast<int>(data.d));
    w.push_back(AnisotropicWeights::from_eta(eta));
    lo = i == 0 ? eta : std::min(lo, eta);
    hi = i == 0 ? eta : std::max(hi, eta);
    sum += eta;
  }
  if (meta) {
    meta->add("threshold", jnum(spec.threshold));
    meta->add("derived_eta_min", jnum(lo));
    meta->add("derived_eta_mean", jnum(sum / static_cast<double>(data.n)));
    meta->add("derived_eta_max", jnum(hi));
  }
  return w;
}

std::string policy_defaults() {
  Doc q;
  q.add("abs_tol", jnum(1e-10)).add("rel_tol", jnum(1e-12)).add("max_depth", jint(40));
  Doc d;
  d.add("tie_break", jstr("lowest_index"))
      .add("empty_partition_policy", jstr("reseed_highest_loss"))
      .add("ridge_vq_default", jstr("1e-10 * mean h_perp"))
      .add("ridge_pq_default", jstr("1e-6 * trace / unknowns"))
      .add("assignment_sweeps", jstr("one fixed-order pass per iteration"))
      .add("eta_derivation", jstr("large-d limit proxy of the indicator weight"))
      .add("quadrature", q.dump());
  return d.dump();
}

anisoq::Dataset load_dataset(const std::string& path, bool normalize) {
  anisoq::Dataset ds = anisoq::read_fvecs(path);
  if (normalize) ds = anisoq::unit_normalize(ds);
  return ds;
}

std::string digest_entry(const std::string& path) {
  Doc d;
  d.add("path", jstr(path)).add("fnv1a64", jstr(file_digest(path)));
  return d.dump();
}

int run_gen(int argc, char** argv) {
  std::string out, kind = "uniform_sphere";
  std::size_t n = 1000, d = 16, centers = 16;
  std::uint64_t seed = 0;
  double spread = 0.25;
  bool normalize = false;
  Verb v{"gen", {}, {}};
  v.opt("out", out, true);
  v.opt("kind", kind);
  v.opt("n", n);
  v.opt("d", d);
  v.opt("seed", seed);
  v.opt("centers", centers);
  v.opt("spread", spread);
  v.flag("normalize", normalize);
  v.parse(argc, argv, 2);
  v.check_required();
  v.apply_config();
  anisoq::SyntheticParams params;
  params.centers = centers;
  params.spread = spread;
  params.normalize = normalize;
  const anisoq::SyntheticKind k =
      kind == "uniform_sphere"     ? anisoq::SyntheticKind::uniform_sphere
      : kind == "gaussian_mixture" ? anisoq::SyntheticKind::gaussian_mixture
                                   : throw anisoq::InvalidArgument("unknown kind " + kind);
  const anisoq::Dataset ds = anisoq::generate_synthetic(k, n, d, seed, params);
  anisoq::write_fvecs(ds, out);
  Doc o;
  o.add("out", jstr(out)).add("kind", jstr(kind)).add("n", jint(n)).add("d", jint(d));
  o.add("seed", jint(seed)).add("centers", jint(centers)).add("spread", jnum(spread));
  o.add("normalize", jbool(normalize));
  Doc m;
  m.add("command", jstr("gen")).add("options", o.dump()).add("outputs", jarr({jstr(out)}));
  m.add("output_digest", jstr(file_digest(out)));
  write_json(m, out + ".meta.json");
  std::cout << "wrote " << ds.n << " x " << ds.d << " to " << out << "\n";
  return 0;
}

void write_train_log(const std::string& path, const std::vector<double>& history,
                     const Doc& meta) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw anisoq::MalformedFile("cannot open " + path + " for writing");
  for (const auto& [key, value] : meta.items) out << "# " << key << "=" << value << "\n";
  out << "iteration,total_loss\n";
  char buf[64];
  for (std::size_t i = 0; i < history.size(); ++i) {
    std::snprintf(buf, sizeof(buf), "%zu,%.17g\n", i, history[i]);
    out << buf;
  }
}

int run_train(int argc, char** argv) {
  std::string data, out, quantizer = "pq";
  std::size_t k = 16, M = 8;
  LossSpec loss;
  long iters = 100, threads = 1;
  double tol = 1e-6, ridge = -1.0;
  std::uint64_t seed = 0;
  bool normalize = false, warm_start = true, sweep_fixed = false;
  Verb v{"train", {}, {}};
  v.opt("data", data, true);
  v.opt("out", out, true);
  v.opt("quantizer", quantizer);
  v.opt("k", k);
  v.opt("M", M);
  v.opt("loss", loss.loss);
  v.opt("threshold", loss.threshold);
  v.opt("eta", loss.explicit_eta);
  v.opt("iters", iters);
  v.opt("tol", tol);
  v.opt("seed", seed);
  v.opt("ridge", ridge);
  v.opt("threads", threads);
  v.flag("normalize", normalize);
  v.flag("warm-start", warm_start, true);
  v.flag("sweep-to-fixed-point", sweep_fixed);
  v.parse(argc, argv, 2);
  v.check_required();
  v.apply_config();
  if (quantizer != "vq" && quantizer != "pq")
    throw anisoq::InvalidArgument("quantizer must be vq or pq");
  const anisoq::Dataset ds = load_dataset(data, normalize);
  fs::create_directories(out);
  Doc loss_meta;
  const auto weights = resolve_weights(loss, ds, &loss_meta);
  anisoq::TrainConfig cfg;
  cfg.max_iterations = static_cast<int>(iters);
  cfg.relative_tolerance = tol;
  cfg.seed = seed;
  cfg.ridge = ridge;
  cfg.threads = static_cast<int>(threads);
  cfg.sweep_to_fixed_point = sweep_fixed;

  anisoq::ProductCodebook cb;
  anisoq::CodeMatrix codes;
  std::vector<double> history;
  if (quantizer == "vq") {
    auto [vq_cb, assignment] = anisoq::train_avq(ds, k, weights, cfg);
    cb = anisoq::to_product(vq_cb);
    codes.n = ds.n;
    codes.M = 1;
    codes.k = k;
    codes.codes = assignment.assignments;
    history = assignment.loss_history;
  } else {
    std::tie(cb, codes) = anisoq::train_apq(ds, M, k, weights, cfg, warm_start, &history);
  }
  anisoq::save_codebook(cb, (fs::path(out) / "codebook.bin").string());
  anisoq::save_codes(codes, (fs::path(out) / "codes.bin").string());
  write_train_log((fs::path(out) / "train_log.csv").string(), history, loss_meta);

  Doc o;
  o.add("data", jstr(data)).add("quantizer", jstr(quantizer)).add("k", jint(k));
  o.add("M", jint(quantizer == "pq" ? M : 1)).add("iters", jint(iters)).add("tol", jnum(tol));
  o.add("seed", jint(seed)).add("ridge", jnum(ridge)).add("threads", jint(threads));
  o.add("normalize", jbool(normalize)).add("warm_start", jbool(warm_start));
  o.add("sweep_to_fixed_point", jbool(sweep_fixed));
  Doc in;
  in.add("data", digest_entry(data));
  const double final_loss = history.empty() ? 0.0 : history.back();
  Doc m;
  m.add("command", jstr("train")).add("options", o.dump()).add("loss", loss_meta.dump());
  m.add("inputs", in.dump());
  m.add("outputs", jarr({jstr("codebook.bin"), jstr("codes.bin"), jstr("train_log.csv")}));
  m.add("policies", policy_defaults()).add("final_loss", jnum(final_loss));
  m.add("iterations_run", jint(history.empty() ? 0 : history.size() - 1));
  write_json(m, (fs::path(out) / "manifest.json").string());
  std::cout << "trained " << quantizer << " codebook: k=" << k
            << (quantizer == "pq" ? " M=" + std::to_string(M) : "") << " final_loss=" << final_loss
            << "\n";
  return 0;
}

int run_encode(int argc, char** argv) {
  std::string data, codebook, out;
  LossSpec loss;
  long passes = 1, threads = 1;
  bool normalize = false;
  Verb v{"encode", {}, {}};
  v.opt("data", data, true);
  v.opt("codebook", codebook, true);
  v.opt("out", out, true);
  v.opt("loss", loss.loss);
  v.opt("threshold", loss.threshold);
  v.opt("eta", loss.explicit_eta);
  v.opt("passes", passes);
  v.opt("threads", threads);
  v.flag("normalize", normalize);
  v.parse(argc, argv, 2);
  v.check_required();
  v.apply_config();
  const anisoq::Dataset ds = load_dataset(data, normalize);
  const auto cb = anisoq::load_codebook(codebook);
  Doc loss_meta;
  const auto weights = resolve_weights(loss, ds, &loss_meta);
  const auto codes =
      anisoq::pq_quantize(ds, cb, weights, static_cast<int>(passes), static_cast<int>(threads));
  anisoq::save_codes(codes, out);
  Doc o;
  o.add("data", jstr(data)).add("codebook", jstr(codebook)).add("out", jstr(out));
  o.add("passes", jint(passes)).add("threads", jint(threads)).add("normalize", jbool(normalize));
  Doc in;
  in.add("data", digest_entry(data)).add("codebook", digest_entry(codebook));
  Doc m;
  m.add("command", jstr("encode")).add("options", o.dump()).add("loss", loss_meta.dump());
  m.add("inputs", in.dump()).add("outputs", jarr({jstr(out)}));
  write_json(m, out + ".meta.json");
  std::cout << "encoded " << codes.n << " datapoints\n";
  return 0;
}

int run_search(int argc, char** argv) {
  std::string codebook, codes_path, queries_path;
  std::size_t topn = 10;
  long query_index = -1;
  bool normalize = false;
  Verb v{"search", {}, {}};
  v.opt("codebook", codebook, true);
  v.opt("codes", codes_path, true);
  v.opt("queries", queries_path, true);
  v.opt("topn", topn);
  v.opt("query-index", query_index);
  v.flag("normalize", normalize);
  v.parse(argc, argv, 2);
  v.check_required();
  v.apply_config();
  const auto cb = anisoq::load_codebook(codebook);
  const auto codes = anisoq::load_codes(codes_path);
  const anisoq::Dataset queries = load_dataset(queries_path, normalize);
  if (queries.n == 0) throw anisoq::EmptyDataset("no queries in " + queries_path);
  const std::size_t begin = query_index >= 0 ? static_cast<std::size_t>(query_index) : 0;
  const std::size_t end = query_index >= 0 ? begin + 1 : queries.n;
  if (begin >= queries.n) throw anisoq::InvalidArgument("query index out of range");
  // all queries of the range as one device batch (adc_search per query,
  // index.hpp:118-134, bit for bit)
  const std::size_t nq = end - begin, keep = std::min(topn, codes.n);
  if (queries.d != cb.dim()) throw anisoq::DimensionMismatch("query dimension does not match codebook");
  std::vector<std::uint32_t> ids(nq * keep);
  std::vector<double> scores(nq * keep);
  anisoq::b200::check(aq_adc_search_batch(
      anisoq::b200::session(), queries.values.data() + begin * queries.d, nq, queries.d,
      codes.codes.data(), codes.n, codes.M, codes.k, cb.dictionaries.data(), cb.M, cb.k,
      cb.sub_dimension, topn, ids.data(), scores.data()));
  std::cout << "# query rank index score\n";
  char buf[96];
  for (std::size_t q = 0; q < nq; ++q)
    for (std::size_t r = 0; r < keep; ++r) {
      std::snprintf(buf, sizeof(buf), "%zu %zu %u %.9g\n", begin + q, r, ids[q * keep + r],
                    scores[q * keep + r]);
      std::cout << buf;
    }
  return 0;
}

std::vector<std::size_t> parse_ns(const std::string& text) {
  std::vector<std::size_t> ns;
  std::stringstream ss(text);
  std::string item;
  while (std::getline(ss, item, ',')) {
    if (item.empty()) continue;
    ns.push_back(static_cast<std::size_t>(std::stoull(item)));
  }
  if (ns.empty()) throw anisoq::InvalidArgument("empty N list");
  return ns;
}

int run_eval(int argc, char** argv) {
  std::string data, queries_path, codebook, codes_path, out, ns = "1,10,100", ground_truth;
  std::size_t kk = 10;
  long threads = 1;
  bool normalize = false;
  Verb v{"eval", {}, {}};
  v.opt("data", data, true);
  v.opt("queries", queries_path, true);
  v.opt("codebook", codebook, true);
  v.opt("codes", codes_path, true);
  v.opt("out", out, true);
  v.opt("Ns", ns);
  v.opt("kk", kk);
  v.opt("ground-truth", ground_truth);
  v.opt("threads", threads);
  v.flag("normalize", normalize);
  v.parse(argc, argv, 2);
  v.check_required();
  v.apply_config();
  const anisoq::Dataset ds = load_dataset(data, normalize);
  const anisoq::Dataset queries = load_dataset(queries_path, normalize);
  if (queries.n == 0) throw anisoq::EmptyDataset("no queries in " + queries_path);
  const auto cb = anisoq::load_codebook(codebook);
  const auto codes = anisoq::load_codes(codes_path);
  fs::create_directories(out);

  anisoq::EvalOptions opt;
  opt.recall_ns = parse_ns(ns);
  opt.kk = kk;
  opt.threads = static_cast<int>(threads);
  std::size_t depth = opt.kk;
  for (auto n : opt.recall_ns) depth = std::max(depth, n);
  depth = std::min(depth, ds.n);

  const std::string data_digest = file_digest(data), query_digest = file_digest(queries_path);
  std::string gt_path = ground_truth, gt_source;
  std::vector<std::vector<std::int32_t>> gt;
  if (gt_path.empty()) {
    gt_path = (fs::path(out) / ("gt-" + data_digest.substr(0, 12) + "-" +
                                query_digest.substr(0, 12) + "-g" + std::to_string(depth) +
                                ".ivecs"))
                  .string();
    if (fs::exists(gt_path)) {
      gt = anisoq::read_ivecs(gt_path);
      gt_source = "cache";
      if (gt.size() != queries.n || (depth > 0 && (gt.empty() || gt[0].size() < depth)))
        gt.clear();  // stale cache, recomputed below
    }
    if (gt.empty()) {
      gt = anisoq::exact_ground_truth(queries, ds, depth, opt.threads);
      anisoq::write_ivecs(gt, gt_path);
      gt_source = "computed";
    }
  } else if (fs::exists(gt_path)) {
    gt = anisoq::read_ivecs(gt_path);
    gt_source = "supplied";
  } else {
    gt = anisoq::exact_ground_truth(queries, ds, depth, opt.threads);
    anisoq::write_ivecs(gt, gt_path);
    gt_source = "computed";
  }
  opt.ground_truth = &gt;
  const auto report = anisoq::evaluate(queries, ds, codes, cb, opt);
  {
    std::ofstream txt((fs::path(out) / "eval_report.txt").string(), std::ios::trunc);
    report.write_text(txt);
  }
  report.write_text(std::cout);

  Doc rel, lat, r1;
  rel.add("mean", jnum(report.relative_error_mean)).add("p50", jnum(report.relative_error_p50));
  rel.add("p90", jnum(report.relative_error_p90)).add("p99", jnum(report.relative_error_p99));
  rel.add("max", jnum(report.relative_error_max));
  lat.add("mean", jnum(report.latency.mean_us)).add("p50", jnum(report.latency.p50_us));
  lat.add("p99", jnum(report.latency.p99_us));
  for (const auto& [n, r] : report.recall_1_at_n) r1.add(std::to_string(n), jnum(r));
  Doc doc;
  doc.add("kk", jint(report.kk)).add("latency_us", lat.dump());
  doc.add("num_datapoints", jint(report.num_datapoints)).add("num_queries", jint(report.num_queries));
  doc.add("recall_1_at_n", r1.dump()).add("recall_kk", jnum(report.recall_k_at_k));
  doc.add("relative_error_top1", rel.dump());
  write_json(doc, (fs::path(out) / "eval_report.json").string());

  Doc o;
  o.add("data", jstr(data)).add("queries", jstr(queries_path)).add("codebook", jstr(codebook));
  o.add("codes", jstr(codes_path)).add("Ns", jstr(ns)).add("kk", jint(kk));
  o.add("threads", jint(threads)).add("normalize", jbool(normalize));
  Doc in, dd, qd;
  dd.add("path", jstr(data)).add("fnv1a64", jstr(data_digest));
  qd.add("path", jstr(queries_path)).add("fnv1a64", jstr(query_digest));
  in.add("data", dd.dump()).add("queries", qd.dump()).add("codebook", digest_entry(codebook));
  in.add("codes", digest_entry(codes_path));
  Doc g;
  g.add("path", jstr(gt_path)).add("source", jstr(gt_source));
  Doc m;
  m.add("command", jstr("eval")).add("options", o.dump()).add("inputs", in.dump());
  m.add("ground_truth", g.dump());
  m.add("outputs", jarr({jstr("eval_report.txt"), jstr("eval_report.json")}));
  write_json(m, (fs::path(out) / "manifest.json").string());
  return 0;
}

void usage(std::ostream& o) {
  o << "anisotropic (score-aware) quantization toolkit for maximum inner product search "
       "(B200)\nUsage: anisoq_b200 <gen|train|encode|search|eval> [--option value ...]\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
    usage(argc < 2 ? std::cerr : std::cout);
    return argc < 2 ? kExitValidation : 0;
  }
  const std::string verb = argv[1];
  try {
    if (verb == "gen") return run_gen(argc, argv);
    if (verb == "train") return run_train(argc, argv);
    if (verb == "encode") return run_encode(argc, argv);
    if (verb == "search") return run_search(argc, argv);
    if (verb == "eval") return run_eval(argc, argv);
    if (verb == "convert" || verb == "diagnose" || verb == "eta")
      throw anisoq::InvalidArgument(verb + " is not part of the B200 hot path (use the reference tool)");
    throw anisoq::InvalidArgument("unknown subcommand " + verb);
  } catch (const anisoq::Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return e.error_class() == anisoq::ErrorClass::validation ? kExitValidation : kExitRuntime;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitRuntime;
  }
}
