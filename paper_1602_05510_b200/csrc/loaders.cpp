// loaders.cpp — the reference's fixture formats read in C++ (SURVEY.md §8f
// row f4), so a C/C++ caller without the reference can create an engine
// from the same files:
//   Platform::from_json              platform.cpp:157-196
//   PerfModel::from_analytic_json    platform.cpp:305-320
//   PerfModel::from_table_csv        platform.cpp:238-290
// A small JSON reader covers the documents' grammar (objects, arrays,
// strings, numbers, true/false/null); numbers go through strtod/strtoll, which
// round exactly like nlohmann::json.  Parse errors carry the reference's
// wording class (`platform document:` / `analytic model:` / `perf table ...`).
// Validation beyond parsing (ids, main space, routes) is hesp_engine_create's.
#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "hesp_engine.h"
#include "problem.h"

namespace {

struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } k = Null;
  bool b = false;
  std::string num;  // the literal, converted on use
  std::string s;
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;
  const JVal* get(const std::string& key) const {
    for (const auto& kv : o)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  const JVal& at(const std::string& key) const {
    const JVal* v = get(key);
    if (!v) throw std::runtime_error("key '" + key + "' not found");
    return *v;
  }
  double as_double() const {
    if (k != Num) throw std::runtime_error("number expected");
    return std::strtod(num.c_str(), nullptr);
  }
  long long as_int() const {
    if (k != Num) throw std::runtime_error("integer expected");
    if (num.find_first_of(".eE") != std::string::npos) {
      const double d = std::strtod(num.c_str(), nullptr);
      if (d != (double)(long long)d) throw std::runtime_error("integer expected");
      return (long long)d;
    }
    errno = 0;
    const long long v = std::strtoll(num.c_str(), nullptr, 10);
    if (errno) throw std::runtime_error("integer out of range");
    return v;
  }
  const std::string& as_str() const {
    if (k != Str) throw std::runtime_error("string expected");
    return s;
  }
};

struct JParser {
  const std::string& t;
  size_t i = 0;
  void ws() {
    while (i < t.size() && (t[i] == ' ' || t[i] == '\n' || t[i] == '\r' || t[i] == '\t')) ++i;
  }
  [[noreturn]] void bad(const char* what) {
    throw std::runtime_error(std::string("parse error at byte ") + std::to_string(i) + ": " + what);
  }
  JVal value() {
    ws();
    if (i >= t.size()) bad("unexpected end");
    const char c = t[i];
    JVal v;
    if (c == '{') {
      v.k = JVal::Obj;
      ++i;
      ws();
      if (i < t.size() && t[i] == '}') {
        ++i;
        return v;
      }
      for (;;) {
        ws();
        JVal key = value();
        if (key.k != JVal::Str) bad("object key must be a string");
        ws();
        if (i >= t.size() || t[i] != ':') bad("':' expected");
        ++i;
        v.o.emplace_back(key.s, value());
        ws();
        if (i < t.size() && t[i] == ',') {
          ++i;
          continue;
        }
        if (i < t.size() && t[i] == '}') {
          ++i;
          return v;
        }
        bad("',' or '}' expected");
      }
    }
    if (c == '[') {
      v.k = JVal::Arr;
      ++i;
      ws();
      if (i < t.size() && t[i] == ']') {
        ++i;
        return v;
      }
      for (;;) {
        v.a.push_back(value());
        ws();
        if (i < t.size() && t[i] == ',') {
          ++i;
          continue;
        }
        if (i < t.size() && t[i] == ']') {
          ++i;
          return v;
        }
        bad("',' or ']' expected");
      }
    }
    if (c == '"') {
      v.k = JVal::Str;
      ++i;
      while (i < t.size() && t[i] != '"') {
        if (t[i] == '\\') {
          if (++i >= t.size()) bad("bad escape");
          const char e = t[i];
          if (e == 'n') v.s += '\n';
          else if (e == 't') v.s += '\t';
          else if (e == 'r') v.s += '\r';
          else if (e == 'b') v.s += '\b';
          else if (e == 'f') v.s += '\f';
          else if (e == 'u') {  // fixtures use ASCII; keep \u escapes verbatim
            v.s += "\\u";
          } else v.s += e;
          ++i;
          continue;
        }
        v.s += t[i++];
      }
      if (i >= t.size()) bad("unterminated string");
      ++i;
      return v;
    }
    if (t.compare(i, 4, "true") == 0) {
      i += 4;
      v.k = JVal::Bool;
      v.b = true;
      return v;
    }
    if (t.compare(i, 5, "false") == 0) {
      i += 5;
      v.k = JVal::Bool;
      return v;
    }
    if (t.compare(i, 4, "null") == 0) {
      i += 4;
      return v;
    }
    const size_t s0 = i;
    if (t[i] == '-') ++i;
    while (i < t.size() && (std::isdigit((unsigned char)t[i]) || t[i] == '.' || t[i] == 'e' || t[i] == 'E' ||
                            t[i] == '+' || t[i] == '-'))
      ++i;
    if (i == s0) bad("value expected");
    v.k = JVal::Num;
    v.num = t.substr(s0, i - s0);
    return v;
  }
  JVal document() {
    JVal v = value();
    ws();
    if (i != t.size()) bad("trailing characters");
    return v;
  }
};

std::string slurp(const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error(std::string("cannot open ") + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

int kind_from(const std::string& s) {  // task_kind_from, platform.cpp:49-55
  if (s == "CHOL") return HESP_CHOL;
  if (s == "TRSM") return HESP_TRSM;
  if (s == "SYRK") return HESP_SYRK;
  if (s == "GEMM") return HESP_GEMM;
  throw std::runtime_error("unknown task kind '" + s + "'");
}

std::vector<std::string> split_csv(const std::string& line) {  // split_csv_line, platform.cpp:227-236
  std::vector<std::string> out;
  std::stringstream ss(line);
  std::string f;
  while (std::getline(ss, f, ',')) {
    const auto b = f.find_first_not_of(" \t\r");
    const auto e = f.find_last_not_of(" \t\r");
    out.push_back(b == std::string::npos ? "" : f.substr(b, e - b + 1));
  }
  return out;
}

}  // namespace

struct hesp_fixture {
  std::vector<hesp_space> spaces;
  std::vector<std::string> type_names;
  std::vector<const char*> type_ptrs;
  std::vector<hesp_processor> procs;
  std::vector<hesp_link> links;
  std::vector<hesp_analytic_entry> entries;
  std::vector<hesp_table_row> rows;
  hesp_platform platform{};
  hesp_perf_model model{};
};

extern "C" {

hesp_fixture* hesp_fixture_load(const char* platform_path, const char* model_path) {
  if (!platform_path || !model_path) {
    hx::set_last_error("hesp_fixture_load: null path");
    return nullptr;
  }
  std::unique_ptr<hesp_fixture> fx(new hesp_fixture());
  std::map<std::string, int> tix;
  try {  // Platform::from_json
    std::string text = slurp(platform_path);
    JVal doc;
    try {
      doc = JParser{text}.document();
      for (const auto& js : doc.at("spaces").a) {
        const JVal* m = js.get("is_main");
        fx->spaces.push_back({(int32_t)js.at("id").as_int(), (int64_t)js.at("capacity_bytes").as_int(),
                              m && m->k == JVal::Bool && m->b ? 1 : 0});
      }
      for (const auto& jt : doc.at("types").a) {
        tix[jt.at("name").as_str()] = (int)fx->type_names.size();
        fx->type_names.push_back(jt.at("name").as_str());
      }
      for (const auto& jp : doc.at("processors").a) {
        const std::string tn = jp.at("type").as_str();
        if (!tix.count(tn)) throw std::invalid_argument("processor references unknown type '" + tn + "'");
        fx->procs.push_back({(int32_t)jp.at("id").as_int(), tix[tn], (int32_t)jp.at("space").as_int()});
      }
      if (const JVal* jl = doc.get("links"))
        for (const auto& l : jl->a)
          fx->links.push_back({(int32_t)l.at("src").as_int(), (int32_t)l.at("dst").as_int(),
                               l.at("latency_s").as_double(), l.at("bandwidth_Bps").as_double()});
    } catch (const std::invalid_argument& e) {
      throw std::runtime_error(e.what());
    } catch (const std::runtime_error& e) {
      throw std::runtime_error(std::string("platform document: ") + e.what());
    }
  } catch (const std::exception& e) {
    hx::set_last_error(e.what());
    return nullptr;
  }
  try {
    const std::string mp = model_path;
    const bool csv = mp.size() >= 4 && mp.compare(mp.size() - 4, 4, ".csv") == 0;
    std::string text = slurp(model_path);
    if (!csv) {  // PerfModel::from_analytic_json (+ analytic's validation)
      JVal doc;
      try {
        doc = JParser{text}.document();
        for (const auto& je : doc.a) {
          const int kind = kind_from(je.at("kind").as_str());
          const std::string ty = je.at("proc_type").as_str();
          const double peak = je.at("peak_flops").as_double(), bh = je.at("b_half").as_double();
          if (peak <= 0) throw std::invalid_argument("analytic model: peak_flops must be positive");
          if (bh <= 0) throw std::invalid_argument("analytic model: b_half must be positive");
          auto it = tix.find(ty);
          if (it != tix.end()) fx->entries.push_back({kind, it->second, peak, bh});  // other types: unused
        }
      } catch (const std::invalid_argument& e) {
        throw std::runtime_error(e.what());
      } catch (const std::runtime_error& e) {
        throw std::runtime_error(std::string("analytic model: ") + e.what());
      }
      fx->model.variant = HESP_MODEL_ANALYTIC;
    } else {  // PerfModel::from_table_csv
      std::stringstream ss(text);
      std::string line;
      bool header = false;
      int lineno = 0;
      while (std::getline(ss, line)) {
        ++lineno;
        auto f = split_csv(line);
        if (f.empty() || (f.size() == 1 && f[0].empty())) continue;
        if (!header) {
          if (f != std::vector<std::string>{"kind", "proc_type", "b", "seconds"})
            throw std::runtime_error("perf table: expected header kind,proc_type,b,seconds");
          header = true;
          continue;
        }
        if (f.size() != 4) throw std::runtime_error("perf table line " + std::to_string(lineno) + ": expected 4 fields");
        const int kind = kind_from(f[0]);
        char* e1 = nullptr;
        char* e2 = nullptr;
        const long long b = std::strtoll(f[2].c_str(), &e1, 10);
        const double sec = std::strtod(f[3].c_str(), &e2);
        if (e1 == f[2].c_str() || e2 == f[3].c_str())
          throw std::runtime_error("perf table line " + std::to_string(lineno) + ": bad number");
        if (b < 1) throw std::runtime_error("perf table line " + std::to_string(lineno) + ": b must be >= 1");
        if (sec <= 0) throw std::runtime_error("perf table line " + std::to_string(lineno) + ": nonpositive time");
        auto it = tix.find(f[1]);
        if (it != tix.end()) fx->rows.push_back({kind, it->second, b, sec});
      }
      fx->model.variant = HESP_MODEL_TABULATED;
    }
  } catch (const std::exception& e) {
    hx::set_last_error(e.what());
    return nullptr;
  }
  for (const auto& n : fx->type_names) fx->type_ptrs.push_back(n.c_str());
  fx->platform = hesp_platform{(int32_t)fx->spaces.size(), fx->spaces.data(), (int32_t)fx->type_ptrs.size(),
                               fx->type_ptrs.data(), (int32_t)fx->procs.size(), fx->procs.data(),
                               (int32_t)fx->links.size(), fx->links.data()};
  fx->model.n_entries = (int32_t)fx->entries.size();
  fx->model.entries = fx->entries.data();
  fx->model.n_rows = (int32_t)fx->rows.size();
  fx->model.rows = fx->rows.data();
  return fx.release();
}

const hesp_platform* hesp_fixture_platform(const hesp_fixture* f) { return f ? &f->platform : nullptr; }
const hesp_perf_model* hesp_fixture_model(const hesp_fixture* f) { return f ? &f->model : nullptr; }
void hesp_fixture_free(hesp_fixture* f) { delete f; }

}  // extern "C"
