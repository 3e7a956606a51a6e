// Action-list JSON: byte-compatible writer and strict reader.
//
// The on-disk format of the reference goldens (src/serialize.cpp:236-307):
// an object {"config", "placement", "actions"} pretty-printed the way stock
// nlohmann::ordered_json::dump(2) prints it -- two-space indent, one element
// per line, "[]" / "{}" for empty containers, trailing newline.  The reader
// enforces the same schema rules as src/serialize.cpp:79-232 (unknown fields,
// enum names, ranges, placement shape) and reports the offending location.
// Self-contained: no third-party JSON library.
#include <cctype>
#include <cstring>
#include <map>
#include <memory>
#include <set>

#include "wavepipe/core.hpp"

namespace wavepipe {

namespace {

// ---------------------------------------------------------------- value tree
struct JVal {
  enum T { Null, Bool, Int, Float, Str, Arr, Obj } t = Null;
  bool b = false;
  int64_t i = 0;
  double f = 0;
  std::string s;
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;  // insertion ordered

  const JVal* get(const std::string& k) const {
    for (const auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

[[noreturn]] void fail(const std::string& where, const std::string& what) {
  throw ParseError(where + ": " + what);
}

class Reader {
 public:
  explicit Reader(const std::string& t) : p_(t.data()), e_(t.data() + t.size()) {}
  JVal parse_document() {
    JVal v = value();
    ws();
    if (p_ != e_) bad("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void bad(const char* why) { throw ParseError(std::string("invalid JSON: ") + why); }
  void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (size_t(e_ - p_) >= n && std::memcmp(p_, w, n) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  JVal value() {
    ws();
    if (p_ >= e_) bad("unexpected end of input");
    JVal v;
    switch (*p_) {
      case '{': {
        ++p_;
        v.t = JVal::Obj;
        ws();
        if (p_ < e_ && *p_ == '}') { ++p_; return v; }
        for (;;) {
          ws();
          if (p_ >= e_ || *p_ != '"') bad("expected object key");
          std::string k = str();
          ws();
          if (p_ >= e_ || *p_ != ':') bad("expected ':'");
          ++p_;
          JVal child = value();
          bool replaced = false;
          for (auto& kv : v.o)
            if (kv.first == k) { kv.second = child; replaced = true; }
          if (!replaced) v.o.emplace_back(std::move(k), std::move(child));
          ws();
          if (p_ < e_ && *p_ == ',') { ++p_; continue; }
          if (p_ < e_ && *p_ == '}') { ++p_; return v; }
          bad("expected ',' or '}'");
        }
      }
      case '[': {
        ++p_;
        v.t = JVal::Arr;
        ws();
        if (p_ < e_ && *p_ == ']') { ++p_; return v; }
        for (;;) {
          v.a.push_back(value());
          ws();
          if (p_ < e_ && *p_ == ',') { ++p_; continue; }
          if (p_ < e_ && *p_ == ']') { ++p_; return v; }
          bad("expected ',' or ']'");
        }
      }
      case '"':
        v.t = JVal::Str;
        v.s = str();
        return v;
      default:
        break;
    }
    if (lit("true")) { v.t = JVal::Bool; v.b = true; return v; }
    if (lit("false")) { v.t = JVal::Bool; return v; }
    if (lit("null")) return v;
    return number();
  }
  std::string str() {
    ++p_;  // opening quote
    std::string out;
    while (p_ < e_ && *p_ != '"') {
      if (static_cast<unsigned char>(*p_) < 0x20) bad("control character in string");
      if (*p_ != '\\') { out += *p_++; continue; }
      if (++p_ >= e_) bad("bad escape");
      const char c = *p_++;
      switch (c) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          if (e_ - p_ < 4) bad("bad unicode escape");
          unsigned cp = std::stoul(std::string(p_, 4), nullptr, 16);
          p_ += 4;
          if (cp < 0x80) out += char(cp);
          else if (cp < 0x800) { out += char(0xC0 | (cp >> 6)); out += char(0x80 | (cp & 0x3F)); }
          else { out += char(0xE0 | (cp >> 12)); out += char(0x80 | ((cp >> 6) & 0x3F)); out += char(0x80 | (cp & 0x3F)); }
          break;
        }
        default: bad("bad escape");
      }
    }
    if (p_ >= e_) bad("unterminated string");
    ++p_;
    return out;
  }
  JVal number() {
    const char* b = p_;
    if (p_ < e_ && *p_ == '-') ++p_;
    if (p_ >= e_ || !std::isdigit(static_cast<unsigned char>(*p_))) bad("unexpected character");
    if (*p_ == '0') ++p_;
    else while (p_ < e_ && std::isdigit(static_cast<unsigned char>(*p_))) ++p_;
    bool integral = true;
    if (p_ < e_ && *p_ == '.') {
      integral = false;
      ++p_;
      if (p_ >= e_ || !std::isdigit(static_cast<unsigned char>(*p_))) bad("bad number");
      while (p_ < e_ && std::isdigit(static_cast<unsigned char>(*p_))) ++p_;
    }
    if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
      integral = false;
      ++p_;
      if (p_ < e_ && (*p_ == '+' || *p_ == '-')) ++p_;
      if (p_ >= e_ || !std::isdigit(static_cast<unsigned char>(*p_))) bad("bad number");
      while (p_ < e_ && std::isdigit(static_cast<unsigned char>(*p_))) ++p_;
    }
    JVal v;
    const std::string text(b, p_);
    if (integral) {
      errno = 0;
      v.t = JVal::Int;
      v.i = std::strtoll(text.c_str(), nullptr, 10);
      if (errno == ERANGE) { v.t = JVal::Float; v.f = std::strtod(text.c_str(), nullptr); }
    } else {
      v.t = JVal::Float;
      v.f = std::strtod(text.c_str(), nullptr);
    }
    return v;
  }
  const char* p_;
  const char* e_;
};

// ------------------------------------------------------------------- writer
// dump(2) layout of the fixed schema, written directly.
class Writer {
 public:
  std::string out;
  void indent(int n) { out.append(size_t(n) * 2, ' '); }
  void key(int depth, const char* k, bool first) {
    out += first ? "\n" : ",\n";
    indent(depth);
    out += '"';
    out += k;
    out += "\": ";
  }
};

// ------------------------------------------------------------- schema reads
void allow_only(const JVal& obj, const std::string& where, std::initializer_list<const char*> keys) {
  for (const auto& kv : obj.o) {
    bool ok = false;
    for (const char* k : keys) ok = ok || kv.first == k;
    if (!ok) fail(where, "unknown field '" + kv.first + "'");
  }
}

int need_int(const JVal& obj, const std::string& where, const char* k) {
  const JVal* v = obj.get(k);
  if (!v) fail(where, std::string("missing field '") + k + "'");
  if (v->t != JVal::Int) fail(where, std::string("field '") + k + "' must be an integer");
  return static_cast<int>(v->i);
}

std::string need_str(const JVal& obj, const std::string& where, const char* k) {
  const JVal* v = obj.get(k);
  if (!v) fail(where, std::string("missing field '") + k + "'");
  if (v->t != JVal::Str) fail(where, std::string("field '") + k + "' must be a string");
  return v->s;
}

}  // namespace

std::string serialize_action_list(const ActionList& list) {
  Writer w;
  const ScheduleConfig& c = list.config;
  w.out = "{";
  w.key(1, "config", true);
  w.out += "{";
  w.key(2, "scheme", true);
  w.out += std::string("\"") + scheme_name(c.scheme) + "\"";
  const std::pair<const char*, int> nums[] = {{"P", c.devices}, {"B", c.microbatches},
                                              {"W", c.waves}, {"D", c.replicas}, {"S", c.stages}};
  for (const auto& kv : nums) {
    w.key(2, kv.first, false);
    w.out += std::to_string(kv.second);
  }
  w.out += "\n  }";

  w.key(1, "placement", false);
  const auto& as = list.placement.assignment;
  if (as.empty()) w.out += "[]";
  else {
    w.out += "[";
    for (size_t d = 0; d < as.size(); ++d) {
      w.out += d ? ",\n    " : "\n    ";
      if (as[d].empty()) { w.out += "[]"; continue; }
      w.out += "[";
      for (size_t i = 0; i < as[d].size(); ++i) {
        const StageSlice& sl = as[d][i];
        w.out += i ? ",\n      {" : "\n      {";
        w.key(4, "index", true);
        w.out += std::to_string(sl.index);
        w.key(4, "fraction", false);
        w.out += "[\n          " + std::to_string(sl.fraction.num()) + ",\n          " +
                 std::to_string(sl.fraction.den()) + "\n        ]";
        w.key(4, "direction", false);
        w.out += std::string("\"") + direction_name(sl.direction) + "\"\n      }";
      }
      w.out += "\n    ]";
    }
    w.out += "\n  ]";
  }

  w.key(1, "actions", false);
  const auto& pd = list.per_device;
  if (pd.empty()) w.out += "[]";
  else {
    w.out += "[";
    for (size_t d = 0; d < pd.size(); ++d) {
      w.out += d ? ",\n    " : "\n    ";
      if (pd[d].empty()) { w.out += "[]"; continue; }
      w.out += "[";
      for (size_t i = 0; i < pd[d].size(); ++i) {
        const Action& a = pd[d][i];
        w.out += i ? ",\n      {" : "\n      {";
        w.key(4, "kind", true);
        w.out += std::string("\"") + action_kind_name(a.kind) + "\"";
        const std::pair<const char*, int> f[] = {{"microbatch", a.microbatch},
                                                 {"local_module_rank", a.local_module_rank},
                                                 {"slice_index", a.slice_index},
                                                 {"peer", a.peer}};
        for (const auto& kv : f) {
          if (kv.second < 0) continue;
          w.key(4, kv.first, false);
          w.out += std::to_string(kv.second);
        }
        if (a.payload >= 0) {
          w.key(4, "payload", false);
          w.out += std::string("\"") + payload_name(static_cast<Payload>(a.payload)) + "\"";
        }
        if (a.batch_group >= 0) {
          w.key(4, "batch_group", false);
          w.out += std::to_string(a.batch_group);
        }
        w.out += "\n      }";
      }
      w.out += "\n    ]";
    }
    w.out += "\n  ]";
  }
  w.out += "\n}\n";
  return w.out;
}

ActionList parse_action_list(const std::string& text) {
  const JVal doc = Reader(text).parse_document();
  if (doc.t != JVal::Obj) fail("document", "top level must be an object");
  allow_only(doc, "document", {"config", "placement", "actions"});
  for (const char* k : {"config", "placement", "actions"}) {
    if (!doc.get(k)) fail("document", std::string("missing field '") + k + "'");
  }

  ActionList list;
  // config (ref src/serialize.cpp:147-171)
  {
    const JVal& j = *doc.get("config");
    const std::string where = "config";
    if (j.t != JVal::Obj) fail(where, "must be an object");
    allow_only(j, where, {"scheme", "P", "B", "W", "D", "S"});
    const std::string sname = need_str(j, where, "scheme");
    Scheme scheme;
    if (!scheme_from_name(sname, &scheme)) fail(where, "unknown scheme '" + sname + "'");
    const int P = need_int(j, where, "P"), B = need_int(j, where, "B"), W = need_int(j, where, "W"),
              D = need_int(j, where, "D"), S = need_int(j, where, "S");
    try {
      list.config = make_config(scheme, P, B, W, D);
    } catch (const ConfigError& e) {
      fail(where, e.what());
    }
    if (list.config.stages != S) {
      fail(where, "S must equal " + std::to_string(list.config.stages) + " for this config");
    }
  }
  const ScheduleConfig& cfg = list.config;
  const bool chimera = cfg.scheme == Scheme::Chimera;

  // placement (ref src/serialize.cpp:173-232)
  {
    const JVal& j = *doc.get("placement");
    if (j.t != JVal::Arr || static_cast<int>(j.a.size()) != cfg.devices) {
      fail("placement", "must be an array with one entry per device");
    }
    list.placement.assignment.resize(cfg.devices);
    std::vector<int> seen(size_t(cfg.stages) * (chimera ? 2 : 1), 0);
    const Rational expected = is_wave_scheme(cfg.scheme) ? Rational(1, 2 * cfg.waves) : Rational(1);
    for (int d = 0; d < cfg.devices; ++d) {
      const JVal& dev = j.a[d];
      const std::string dw = "placement[" + std::to_string(d) + "]";
      if (dev.t != JVal::Arr) fail(dw, "must be an array of slices");
      Rational total(0);
      for (size_t i = 0; i < dev.a.size(); ++i) {
        const std::string where = dw + "[" + std::to_string(i) + "]";
        const JVal& sj = dev.a[i];
        if (sj.t != JVal::Obj) fail(where, "slice must be an object");
        allow_only(sj, where, {"index", "fraction", "direction"});
        StageSlice sl;
        sl.index = need_int(sj, where, "index");
        if (sl.index < 0 || sl.index >= cfg.stages) fail(where, "slice index out of range");
        const JVal* fr = sj.get("fraction");
        if (!fr) fail(where, "missing field 'fraction'");
        if (fr->t != JVal::Arr || fr->a.size() != 2 || fr->a[0].t != JVal::Int || fr->a[1].t != JVal::Int) {
          fail(where, "field 'fraction' must be a [numerator, denominator] pair");
        }
        if (fr->a[1].i <= 0) fail(where, "fraction denominator must be positive");
        sl.fraction = Rational(fr->a[0].i, fr->a[1].i);
        const std::string dir = need_str(sj, where, "direction");
        if (!direction_from_name(dir, &sl.direction)) fail(where, "unknown direction '" + dir + "'");
        if (sl.fraction != expected) fail(where, "fraction must be " + expected.to_string() + " for this scheme");
        const int slot = sl.index + ((chimera && sl.direction == Direction::Up) ? cfg.stages : 0);
        if (seen[slot]++) fail(where, "duplicate slice assignment");
        total += sl.fraction;
        list.placement.assignment[d].push_back(sl);
      }
      const Rational want(chimera ? 2 : 1);
      if (total != want) fail(dw, "per-device fractions must sum to " + want.to_string());
    }
    for (size_t slot = 0; slot < seen.size(); ++slot) {
      if (!seen[slot]) {
        fail("placement", "slice " + std::to_string(slot % cfg.stages) + " is not assigned to any device");
      }
    }
  }

  // actions (ref src/serialize.cpp:79-145, 289-305)
  const JVal& acts = *doc.get("actions");
  if (acts.t != JVal::Arr || static_cast<int>(acts.a.size()) != cfg.devices) {
    fail("actions", "must be an array with one entry per device");
  }
  list.per_device.resize(cfg.devices);
  for (int d = 0; d < cfg.devices; ++d) {
    const JVal& dev = acts.a[d];
    if (dev.t != JVal::Arr) fail("actions[" + std::to_string(d) + "]", "must be an array");
    const auto& slices = list.placement.assignment[d];
    for (size_t i = 0; i < dev.a.size(); ++i) {
      const std::string where = "actions[" + std::to_string(d) + "][" + std::to_string(i) + "]";
      const JVal& j = dev.a[i];
      if (j.t != JVal::Obj) fail(where, "action must be an object");
      allow_only(j, where, {"kind", "microbatch", "local_module_rank", "slice_index", "peer", "payload",
                            "batch_group"});
      Action a;
      const std::string kind = need_str(j, where, "kind");
      if (!action_kind_from_name(kind, &a.kind)) fail(where, "unknown action kind '" + kind + "'");
      if (a.kind == ActionKind::OptimizerStep) {
        allow_only(j, where, {"kind"});
        list.per_device[d].push_back(a);
        continue;
      }
      a.microbatch = need_int(j, where, "microbatch");
      if (a.microbatch < 0 || a.microbatch >= cfg.microbatches) fail(where, "microbatch out of range");
      a.local_module_rank = need_int(j, where, "local_module_rank");
      if (a.local_module_rank < 0 || a.local_module_rank >= static_cast<int>(slices.size())) {
        fail(where, "local_module_rank out of range");
      }
      a.slice_index = need_int(j, where, "slice_index");
      if (a.slice_index < 0 || a.slice_index >= cfg.stages) fail(where, "slice_index out of range");
      if (slices[a.local_module_rank].index != a.slice_index) {
        fail(where, "slice_index does not match the slice at local_module_rank");
      }
      if (a.is_comm()) {
        a.peer = need_int(j, where, "peer");
        if (a.peer < 0 || a.peer >= cfg.devices) fail(where, "peer rank out of range");
        if (a.peer == d) fail(where, "peer must differ from the device itself");
        const std::string pl = need_str(j, where, "payload");
        Payload p;
        if (!payload_from_name(pl, &p)) fail(where, "unknown payload '" + pl + "'");
        a.payload = static_cast<int>(p);
        if (a.kind == ActionKind::BatchedExchange) {
          a.batch_group = need_int(j, where, "batch_group");
          if (a.batch_group < 0) fail(where, "batch_group must be nonnegative");
        } else if (j.get("batch_group")) {
          fail(where, "field 'batch_group' is only valid on batched_exchange");
        }
      } else {
        for (const char* k : {"peer", "payload", "batch_group"}) {
          if (j.get(k)) fail(where, std::string("field '") + k + "' is not valid on " + kind);
        }
      }
      list.per_device[d].push_back(a);
    }
  }
  return list;
}

}  // namespace wavepipe
