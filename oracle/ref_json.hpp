// Test-oracle JSON codec (oracle/ only): the text transport between the
// Python tests and the unmodified reference library (ref_capi.cpp). Written
// independently of the product's csrc/host/json.hpp + einsum_json.hpp so a
// bug in the product's (de)serialisation cannot hide behind the same bug in
// the oracle ("common-mode risk in the oracle shim").
//
// Values: null / bool / number / string / array / object. Numbers keep their
// literal text (int64 extents and %.17g doubles round-trip exactly); objects
// are std::map (key order is irrelevant to the Python side); strings handle
// the JSON escapes, \uXXXX only below 0x80 (the transport is ASCII).
#pragma once

#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace oj {

struct Value {
  enum Kind { Null, Bool, Num, Str, Arr, Obj };
  Kind k = Null;
  bool b = false;
  std::string s;  // Str payload, or Num literal
  std::vector<Value> a;
  std::map<std::string, Value> o;

  static Value str(const std::string& x) {
    Value v;
    v.k = Str;
    v.s = x;
    return v;
  }
  static Value num(long long x) {
    Value v;
    v.k = Num;
    v.s = std::to_string(x);
    return v;
  }
  static Value dbl(double x) {
    char t[40];
    std::snprintf(t, sizeof t, "%.17g", x);
    Value v;
    v.k = Num;
    v.s = t;
    return v;
  }
  static Value boolean_(bool x) {
    Value v;
    v.k = Bool;
    v.b = x;
    return v;
  }
  static Value arr() {
    Value v;
    v.k = Arr;
    return v;
  }
  static Value obj() {
    Value v;
    v.k = Obj;
    return v;
  }
  void push(Value v) { a.push_back(std::move(v)); }
  void set(const std::string& key, Value v) { o[key] = std::move(v); }
  // nullptr when absent (optional keys)
  const Value* find(const std::string& key) const {
    if (k != Obj) return nullptr;
    auto it = o.find(key);
    return it == o.end() ? nullptr : &it->second;
  }
  const Value& at(const std::string& key) const {
    auto it = o.find(key);
    if (k != Obj || it == o.end()) throw std::runtime_error("oracle json: no key " + key);
    return it->second;
  }
  long long as_int() const {
    if (k != Num) throw std::runtime_error("oracle json: not a number");
    return std::strtoll(s.c_str(), nullptr, 10);
  }
  double as_double() const {
    if (k != Num) throw std::runtime_error("oracle json: not a number");
    return std::strtod(s.c_str(), nullptr);
  }
  const std::string& as_str() const {
    if (k != Str) throw std::runtime_error("oracle json: not a string");
    return s;
  }
};

namespace detail {

struct Reader {
  const std::string& t;
  size_t i = 0;
  explicit Reader(const std::string& text) : t(text) {}
  [[noreturn]] void fail(const char* what) const {
    throw std::runtime_error(std::string("oracle json: ") + what + " at offset " + std::to_string(i));
  }
  void ws() {
    while (i < t.size() && (t[i] == ' ' || t[i] == '\n' || t[i] == '\t' || t[i] == '\r')) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < t.size() && t[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  void need(char c) {
    if (!eat(c)) fail("unexpected character");
  }
  std::string string_body() {
    need('"');
    std::string out;
    while (true) {
      if (i >= t.size()) fail("unterminated string");
      const char c = t[i++];
      if (c == '"') return out;
      if (c != '\\') {
        out += c;
        continue;
      }
      if (i >= t.size()) fail("bad escape");
      const char e = t[i++];
      switch (e) {
        case 'n': out += '\n'; break;
        case 't': out += '\t'; break;
        case 'r': out += '\r'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'u': {
          if (i + 4 > t.size()) fail("bad \\u escape");
          const long cp = std::strtol(t.substr(i, 4).c_str(), nullptr, 16);
          i += 4;
          if (cp >= 0x80) fail("non-ASCII \\u escape");
          out += static_cast<char>(cp);
          break;
        }
        default: out += e;  // \" \\ \/
      }
    }
  }
  Value value() {
    ws();
    if (i >= t.size()) fail("unexpected end");
    const char c = t[i];
    if (c == '{') {
      ++i;
      Value v = Value::obj();
      if (eat('}')) return v;
      do {
        ws();
        const std::string key = string_body();
        need(':');
        v.o[key] = value();
      } while (eat(','));
      need('}');
      return v;
    }
    if (c == '[') {
      ++i;
      Value v = Value::arr();
      if (eat(']')) return v;
      do v.a.push_back(value());
      while (eat(','));
      need(']');
      return v;
    }
    if (c == '"') return Value::str(string_body());
    if (t.compare(i, 4, "true") == 0) {
      i += 4;
      return Value::boolean_(true);
    }
    if (t.compare(i, 5, "false") == 0) {
      i += 5;
      return Value::boolean_(false);
    }
    if (t.compare(i, 4, "null") == 0) {
      i += 4;
      return Value();
    }
    const size_t j = i;
    while (i < t.size() && (std::isdigit(static_cast<unsigned char>(t[i])) || t[i] == '-' || t[i] == '+' ||
                            t[i] == '.' || t[i] == 'e' || t[i] == 'E'))
      ++i;
    if (i == j) fail("unexpected character");
    Value v;
    v.k = Value::Num;
    v.s = t.substr(j, i - j);
    return v;
  }
};

inline void write_string(const std::string& s, std::string& out) {
  out += '"';
  for (const char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      case '\r': out += "\\r"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char u[8];
          std::snprintf(u, sizeof u, "\\u%04x", static_cast<unsigned>(c));
          out += u;
        } else {
          out += c;
        }
    }
  }
  out += '"';
}

inline void write(const Value& v, std::string& out) {
  switch (v.k) {
    case Value::Null: out += "null"; break;
    case Value::Bool: out += v.b ? "true" : "false"; break;
    case Value::Num: out += v.s; break;
    case Value::Str: write_string(v.s, out); break;
    case Value::Arr: {
      out += '[';
      for (size_t n = 0; n < v.a.size(); ++n) {
        if (n) out += ',';
        write(v.a[n], out);
      }
      out += ']';
      break;
    }
    case Value::Obj: {
      out += '{';
      bool first = true;
      for (const auto& kv : v.o) {
        if (!first) out += ',';
        first = false;
        write_string(kv.first, out);
        out += ':';
        write(kv.second, out);
      }
      out += '}';
      break;
    }
  }
}

}  // namespace detail

inline Value parse(const std::string& text) {
  detail::Reader r(text);
  Value v = r.value();
  r.ws();
  if (r.i != text.size()) r.fail("trailing characters");
  return v;
}

inline std::string dump(const Value& v) {
  std::string out;
  detail::write(v, out);
  return out;
}

}  // namespace oj

// The reference's value types <-> the transport schema the Python side
// speaks: {"i_out": [...], "i_in": [[...]], "args": [[{name, shape, dtype}]]},
// sigma maps as objects, permutations as int arrays. Include after the
// reference headers (uses feinsum::dtype_name / dtype_from_name).
namespace ot {

using feinsum::ArrayMeta;
using feinsum::BatchedEinsum;

inline oj::Value list_to_json(const std::vector<std::string>& l) {
  oj::Value v = oj::Value::arr();
  for (const std::string& x : l) v.push(oj::Value::str(x));
  return v;
}

inline std::vector<std::string> strings_of(const oj::Value& v) {
  std::vector<std::string> l;
  l.reserve(v.a.size());
  for (const oj::Value& x : v.a) l.push_back(x.as_str());
  return l;
}

inline oj::Value einsum_to_json(const BatchedEinsum& e) {
  oj::Value rows = oj::Value::arr();
  for (const std::vector<ArrayMeta>& row : e.args) {
    oj::Value r = oj::Value::arr();
    for (const ArrayMeta& m : row) {
      oj::Value mv = oj::Value::obj();
      mv.set("name", oj::Value::str(m.name));
      oj::Value sh = oj::Value::arr();
      for (const auto d : m.shape) sh.push(oj::Value::num(static_cast<long long>(d)));
      mv.set("shape", sh);
      mv.set("dtype", oj::Value::str(feinsum::dtype_name(m.dtype)));
      r.push(mv);
    }
    rows.push(r);
  }
  oj::Value ins = oj::Value::arr();
  for (const auto& l : e.i_in) ins.push(list_to_json(l));
  oj::Value v = oj::Value::obj();
  v.set("i_out", list_to_json(e.i_out));
  v.set("i_in", ins);
  v.set("args", rows);
  return v;
}

inline BatchedEinsum einsum_from_json(const oj::Value& v) {
  BatchedEinsum e;
  e.i_out = strings_of(v.at("i_out"));
  for (const oj::Value& l : v.at("i_in").a) e.i_in.push_back(strings_of(l));
  for (const oj::Value& r : v.at("args").a) {
    std::vector<ArrayMeta> row;
    for (const oj::Value& mv : r.a) {
      ArrayMeta m;
      m.name = mv.at("name").as_str();
      for (const oj::Value& d : mv.at("shape").a) m.shape.push_back(d.as_int());
      m.dtype = feinsum::dtype_from_name(mv.at("dtype").as_str());
      row.push_back(m);
    }
    e.args.push_back(row);
  }
  return e;
}

inline oj::Value strmap_to_json(const std::map<std::string, std::string>& m) {
  oj::Value v = oj::Value::obj();
  for (const auto& kv : m) v.set(kv.first, oj::Value::str(kv.second));
  return v;
}

inline oj::Value ints_to_json(const std::vector<int>& p) {
  oj::Value v = oj::Value::arr();
  for (const int x : p) v.push(oj::Value::num(x));
  return v;
}

template <class W>
oj::Value witness_to_json(const W& w) {
  oj::Value v = oj::Value::obj();
  v.set("sigma_idx", strmap_to_json(w.sigma_idx));
  v.set("sigma_arg", strmap_to_json(w.sigma_arg));
  v.set("sigma_row", ints_to_json(w.sigma_row));
  v.set("sigma_slot", ints_to_json(w.sigma_slot));
  return v;
}

template <class W>
W witness_from_json(const oj::Value& v) {
  W w;
  for (const auto& kv : v.at("sigma_idx").o) w.sigma_idx[kv.first] = kv.second.as_str();
  for (const auto& kv : v.at("sigma_arg").o) w.sigma_arg[kv.first] = kv.second.as_str();
  for (const oj::Value& x : v.at("sigma_row").a) w.sigma_row.push_back(static_cast<int>(x.as_int()));
  for (const oj::Value& x : v.at("sigma_slot").a) w.sigma_slot.push_back(static_cast<int>(x.as_int()));
  return w;
}

}  // namespace ot
