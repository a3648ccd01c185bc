// Minimal JSON value, reader and writer used as the C-ABI transport for
// structured host objects (batched einsums, witnesses, facts). Only what the
// boundary needs: null/bool/number/string/array/object, UTF-8 passthrough,
// \uXXXX escapes below 0x80. Numbers are kept as their source text so int64
// extents and %.17g doubles survive a round trip unchanged.
#pragma once

#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace fejson {

struct Value {
  enum class T { null, boolean, number, string, array, object };
  T t = T::null;
  bool b = false;
  std::string s;  // string payload, or the number's literal text
  std::vector<Value> a;
  std::vector<std::pair<std::string, Value>> o;  // insertion order kept

  static Value str(std::string v) { Value x; x.t = T::string; x.s = std::move(v); return x; }
  static Value num(std::int64_t v) { Value x; x.t = T::number; x.s = std::to_string(v); return x; }
  static Value dbl(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    Value x; x.t = T::number; x.s = buf; return x;
  }
  static Value boolean_(bool v) { Value x; x.t = T::boolean; x.b = v; return x; }
  static Value arr() { Value x; x.t = T::array; return x; }
  static Value obj() { Value x; x.t = T::object; return x; }

  Value& push(Value v) { a.push_back(std::move(v)); return a.back(); }
  Value& set(const std::string& k, Value v) {
    for (auto& kv : o)
      if (kv.first == k) { kv.second = std::move(v); return kv.second; }
    o.emplace_back(k, std::move(v));
    return o.back().second;
  }
  const Value* find(const std::string& k) const {
    for (const auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Value& at(const std::string& k) const {
    const Value* v = find(k);
    if (!v) throw std::runtime_error("json: missing key \"" + k + "\"");
    return *v;
  }
  std::int64_t as_int() const {
    if (t != T::number) throw std::runtime_error("json: expected a number");
    return std::strtoll(s.c_str(), nullptr, 10);
  }
  double as_double() const {
    if (t != T::number) throw std::runtime_error("json: expected a number");
    return std::strtod(s.c_str(), nullptr);
  }
  const std::string& as_str() const {
    if (t != T::string) throw std::runtime_error("json: expected a string");
    return s;
  }
};

inline void write_string(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      case '\r': out += "\\r"; break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", c);
          out += buf;
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

inline void write(std::string& out, const Value& v) {
  switch (v.t) {
    case Value::T::null: out += "null"; break;
    case Value::T::boolean: out += v.b ? "true" : "false"; break;
    case Value::T::number: out += v.s; break;
    case Value::T::string: write_string(out, v.s); break;
    case Value::T::array:
      out += '[';
      for (size_t i = 0; i < v.a.size(); ++i) {
        if (i) out += ',';
        write(out, v.a[i]);
      }
      out += ']';
      break;
    case Value::T::object:
      out += '{';
      for (size_t i = 0; i < v.o.size(); ++i) {
        if (i) out += ',';
        write_string(out, v.o[i].first);
        out += ':';
        write(out, v.o[i].second);
      }
      out += '}';
      break;
  }
}

inline std::string dump(const Value& v) {
  std::string s;
  write(s, v);
  return s;
}

class Reader {
 public:
  explicit Reader(const std::string& text) : p_(text.c_str()), end_(text.c_str() + text.size()) {}

  Value parse_document() {
    Value v = value();
    ws();
    if (p_ != end_) fail("trailing characters");
    return v;
  }

 private:
  const char* p_;
  const char* end_;

  [[noreturn]] void fail(const char* what) { throw std::runtime_error(std::string("json: ") + what); }
  void ws() {
    while (p_ != end_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\t' || *p_ == '\r')) ++p_;
  }
  bool lit(const char* w) {
    const char* q = p_;
    for (; *w; ++w, ++q)
      if (q == end_ || *q != *w) return false;
    p_ = q;
    return true;
  }
  Value value() {
    ws();
    if (p_ == end_) fail("unexpected end");
    char c = *p_;
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value::str(string());
    if (lit("true")) return Value::boolean_(true);
    if (lit("false")) return Value::boolean_(false);
    if (lit("null")) return Value{};
    return number();
  }
  std::string string() {
    if (*p_ != '"') fail("expected a string");
    ++p_;
    std::string out;
    while (true) {
      if (p_ == end_) fail("unterminated string");
      char c = *p_++;
      if (c == '"') break;
      if (c != '\\') { out += c; continue; }
      if (p_ == end_) fail("bad escape");
      char e = *p_++;
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'n': out += '\n'; break;
        case 't': out += '\t'; break;
        case 'r': out += '\r'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'u': {
          if (end_ - p_ < 4) fail("bad \\u escape");
          unsigned code = static_cast<unsigned>(std::strtoul(std::string(p_, 4).c_str(), nullptr, 16));
          p_ += 4;
          if (code < 0x80) out += static_cast<char>(code);
          else if (code < 0x800) {
            out += static_cast<char>(0xC0 | (code >> 6));
            out += static_cast<char>(0x80 | (code & 0x3F));
          } else {
            out += static_cast<char>(0xE0 | (code >> 12));
            out += static_cast<char>(0x80 | ((code >> 6) & 0x3F));
            out += static_cast<char>(0x80 | (code & 0x3F));
          }
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }
  Value number() {
    const char* s = p_;
    if (p_ != end_ && (*p_ == '-' || *p_ == '+')) ++p_;
    while (p_ != end_ && (std::isdigit(static_cast<unsigned char>(*p_)) || *p_ == '.' || *p_ == 'e' ||
                          *p_ == 'E' || *p_ == '-' || *p_ == '+'))
      ++p_;
    if (p_ == s) fail("unexpected character");
    Value v;
    v.t = Value::T::number;
    v.s.assign(s, p_);
    return v;
  }
  Value array() {
    ++p_;
    Value v = Value::arr();
    ws();
    if (p_ != end_ && *p_ == ']') { ++p_; return v; }
    while (true) {
      v.a.push_back(value());
      ws();
      if (p_ == end_) fail("unterminated array");
      if (*p_ == ',') { ++p_; continue; }
      if (*p_ == ']') { ++p_; return v; }
      fail("expected , or ]");
    }
  }
  Value object() {
    ++p_;
    Value v = Value::obj();
    ws();
    if (p_ != end_ && *p_ == '}') { ++p_; return v; }
    while (true) {
      ws();
      std::string k = string();
      ws();
      if (p_ == end_ || *p_ != ':') fail("expected :");
      ++p_;
      v.o.emplace_back(std::move(k), value());
      ws();
      if (p_ == end_) fail("unterminated object");
      if (*p_ == ',') { ++p_; continue; }
      if (*p_ == '}') { ++p_; return v; }
      fail("expected , or }");
    }
  }
};

inline Value parse(const std::string& text) { return Reader(text).parse_document(); }

}  // namespace fejson
