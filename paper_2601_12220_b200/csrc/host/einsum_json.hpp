// JSON transport for the feinsum value types. Include AFTER the feinsum
// headers: the code only touches public field names (i_out/i_in/args,
// ArrayMeta{name,shape,dtype}, the sigma maps) and dtype_name/dtype_from_name,
// so the same text serialises both this library's types and, in the test
// oracle, the reference's identically named types.
#pragma once

#include "json.hpp"

namespace feinsum {
namespace transport {

inline fejson::Value meta_to_json(const ArrayMeta& m) {
  fejson::Value v = fejson::Value::obj();
  v.set("name", fejson::Value::str(m.name));
  fejson::Value sh = fejson::Value::arr();
  for (auto d : m.shape) sh.push(fejson::Value::num(d));
  v.set("shape", std::move(sh));
  v.set("dtype", fejson::Value::str(dtype_name(m.dtype)));
  return v;
}

inline ArrayMeta meta_from_json(const fejson::Value& v) {
  ArrayMeta m;
  m.name = v.at("name").as_str();
  for (const auto& d : v.at("shape").a) m.shape.push_back(d.as_int());
  m.dtype = dtype_from_name(v.at("dtype").as_str());
  return m;
}

inline fejson::Value list_to_json(const std::vector<std::string>& l) {
  fejson::Value v = fejson::Value::arr();
  for (const auto& s : l) v.push(fejson::Value::str(s));
  return v;
}

inline std::vector<std::string> list_from_json(const fejson::Value& v) {
  std::vector<std::string> l;
  for (const auto& s : v.a) l.push_back(s.as_str());
  return l;
}

inline fejson::Value einsum_to_json(const BatchedEinsum& e) {
  fejson::Value v = fejson::Value::obj();
  v.set("i_out", list_to_json(e.i_out));
  fejson::Value in = fejson::Value::arr();
  for (const auto& l : e.i_in) in.push(list_to_json(l));
  v.set("i_in", std::move(in));
  fejson::Value rows = fejson::Value::arr();
  for (const auto& row : e.args) {
    fejson::Value r = fejson::Value::arr();
    for (const auto& m : row) r.push(meta_to_json(m));
    rows.push(std::move(r));
  }
  v.set("args", std::move(rows));
  return v;
}

inline BatchedEinsum einsum_from_json(const fejson::Value& v) {
  BatchedEinsum e;
  e.i_out = list_from_json(v.at("i_out"));
  for (const auto& l : v.at("i_in").a) e.i_in.push_back(list_from_json(l));
  for (const auto& r : v.at("args").a) {
    std::vector<ArrayMeta> row;
    for (const auto& m : r.a) row.push_back(meta_from_json(m));
    e.args.push_back(std::move(row));
  }
  return e;
}

inline fejson::Value strmap_to_json(const std::map<std::string, std::string>& m) {
  fejson::Value v = fejson::Value::obj();
  for (const auto& [k, x] : m) v.set(k, fejson::Value::str(x));
  return v;
}

inline std::map<std::string, std::string> strmap_from_json(const fejson::Value& v) {
  std::map<std::string, std::string> m;
  for (const auto& [k, x] : v.o) m[k] = x.as_str();
  return m;
}

inline fejson::Value ints_to_json(const std::vector<int>& p) {
  fejson::Value v = fejson::Value::arr();
  for (int x : p) v.push(fejson::Value::num(x));
  return v;
}

inline std::vector<int> ints_from_json(const fejson::Value& v) {
  std::vector<int> p;
  for (const auto& x : v.a) p.push_back(static_cast<int>(x.as_int()));
  return p;
}

template <class W>
fejson::Value witness_to_json(const W& w) {
  fejson::Value v = fejson::Value::obj();
  v.set("sigma_idx", strmap_to_json(w.sigma_idx));
  v.set("sigma_arg", strmap_to_json(w.sigma_arg));
  v.set("sigma_row", ints_to_json(w.sigma_row));
  v.set("sigma_slot", ints_to_json(w.sigma_slot));
  return v;
}

template <class W>
W witness_from_json(const fejson::Value& v) {
  W w;
  w.sigma_idx = strmap_from_json(v.at("sigma_idx"));
  w.sigma_arg = strmap_from_json(v.at("sigma_arg"));
  w.sigma_row = ints_from_json(v.at("sigma_row"));
  w.sigma_slot = ints_from_json(v.at("sigma_slot"));
  return w;
}

}  // namespace transport
}  // namespace feinsum
