// Data model, validation and derived sets. Semantics follow the reference
// proj/src/core.cpp:1-250 (messages and their order are pinned by its tests,
// proj/tests/test_core.cpp:47-118). evaluate() lives in evaluate.cpp (device).
#include <algorithm>
#include <sstream>

#include "feinsum/core.hpp"

namespace feinsum {

namespace {

struct DtypeInfo {
  Dtype t;
  const char* name;
  int bytes;
};

constexpr DtypeInfo kDtypes[] = {
    {Dtype::int8, "int8", 1},         {Dtype::int32, "int32", 4},
    {Dtype::int64, "int64", 8},       {Dtype::float16, "float16", 2},
    {Dtype::float32, "float32", 4},   {Dtype::float64, "float64", 8},
    {Dtype::complex64, "complex64", 8}, {Dtype::complex128, "complex128", 16},
};

const DtypeInfo& info(Dtype t) {
  for (const auto& d : kDtypes)
    if (d.t == t) return d;
  throw error(errc::domain, "bad dtype code");
}

std::string comma_joined(const IndexList& l) {
  std::string s;
  for (size_t i = 0; i < l.size(); ++i) s += (i ? "," : "") + l[i];
  return s;
}

template <class... Parts>
std::string cat(const Parts&... parts) {
  std::ostringstream os;
  (os << ... << parts);
  return os.str();
}

}  // namespace

int dtype_size_bytes(Dtype t) { return info(t).bytes; }
const char* dtype_name(Dtype t) { return info(t).name; }

Dtype dtype_from_name(const std::string& s) {
  for (const auto& d : kDtypes)
    if (s == d.name) return d.t;
  throw error(errc::domain, "unknown dtype: " + s);
}

std::int64_t ArrayMeta::num_elements() const {
  std::int64_t n = 1;
  for (std::int64_t d : shape) n *= d;
  return n;
}

std::vector<std::string> validate(const BatchedEinsum& e) {
  std::vector<std::string> out;
  const int rows = e.b(), slots = e.n();

  // 1. shape of the argument matrix
  if (rows < 1) out.push_back("b must be >= 1 (no rows)");
  if (slots < 1) out.push_back("n must be >= 1 (no operand slots)");
  bool rectangular = true;
  for (int r = 0; r < rows; ++r) {
    const size_t w = e.args[r].size();
    if (w != static_cast<size_t>(slots)) {
      out.push_back(cat("row ", r + 1, " has ", w, " args, expected ", slots));
      rectangular = false;
    }
  }
  if (!rectangular || rows < 1 || slots < 1) return out;

  // 2. names, extents, one metadata per name
  std::map<std::string, const ArrayMeta*> first_decl;
  for (int r = 0; r < rows; ++r) {
    for (int k = 0; k < slots; ++k) {
      const ArrayMeta& a = e.args[r][k];
      if (a.name.empty()) {
        out.push_back(cat("row ", r + 1, " slot ", k + 1, ": array name is empty"));
        continue;
      }
      for (size_t d = 0; d < a.shape.size(); ++d)
        if (a.shape[d] < 1)
          out.push_back(cat("array ", a.name, " axis ", d + 1, " has nonpositive length ", a.shape[d]));
      auto ins = first_decl.insert({a.name, &a});
      if (!ins.second && !(*ins.first->second == a))
        out.push_back(cat("row ", r + 1, " slot ", k + 1, ": array ", a.name,
                          " redeclared with different shape or dtype"));
    }
  }

  // 3. arity of every cell against its slot's index list
  bool arity_ok = true;
  for (int r = 0; r < rows; ++r) {
    for (int k = 0; k < slots; ++k) {
      const ArrayMeta& a = e.args[r][k];
      if (a.dim() == static_cast<int>(e.i_in[k].size())) continue;
      arity_ok = false;
      out.push_back(cat("row ", r + 1, " slot ", k + 1, ": array ", a.name, " has ", a.dim(),
                        " dims but index list (", comma_joined(e.i_in[k]), ") has ",
                        e.i_in[k].size()));
    }
  }

  // 4. empty symbols abort the remaining checks
  for (int k = 0; k < slots; ++k)
    for (const auto& s : e.i_in[k])
      if (s.empty()) {
        out.push_back(cat("slot ", k + 1, ": empty index symbol"));
        return out;
      }

  // 5. one extent per symbol over the whole batch
  if (arity_ok) {
    std::map<std::string, std::int64_t> extent;
    for (int k = 0; k < slots; ++k)
      for (size_t d = 0; d < e.i_in[k].size(); ++d)
        for (int r = 0; r < rows; ++r) {
          const std::string& sym = e.i_in[k][d];
          const std::int64_t len = e.args[r][k].shape[d];
          auto ins = extent.insert({sym, len});
          if (!ins.second && ins.first->second != len)
            out.push_back(cat("row ", r + 1, " slot ", k + 1, ": index ", sym, " length mismatch (",
                              ins.first->second, " vs ", len, ")"));
        }
  }

  // 6. output list: nonempty, distinct, read by some slot
  std::set<std::string> read;
  for (const auto& l : e.i_in) read.insert(l.begin(), l.end());
  std::set<std::string> emitted;
  for (const auto& s : e.i_out) {
    if (s.empty()) {
      out.push_back("empty output index symbol");
      continue;
    }
    if (!emitted.insert(s).second) out.push_back("duplicate output index " + s);
    if (read.find(s) == read.end()) out.push_back("output index " + s + " not found in any input");
  }
  return out;
}

void require_valid(const BatchedEinsum& e) {
  const auto problems = validate(e);
  if (problems.empty()) return;
  std::string msg = "invalid batched einsum:";
  for (const auto& p : problems) msg += "\n  " + p;
  throw error(errc::domain, msg);
}

bool equals(const BatchedEinsum& a, const BatchedEinsum& b) { return a == b; }

std::vector<ArrayMeta> universe(const BatchedEinsum& e) {
  std::map<std::string, const ArrayMeta*> by_name;
  for (const auto& row : e.args)
    for (const auto& a : row) by_name.insert({a.name, &a});
  std::vector<ArrayMeta> out;
  out.reserve(by_name.size());
  for (const auto& kv : by_name) out.push_back(*kv.second);
  return out;
}

std::vector<std::string> all_indices(const BatchedEinsum& e) {
  std::vector<std::string> order;
  std::set<std::string> seen;
  for (const auto& l : e.i_in)
    for (const auto& s : l)
      if (seen.insert(s).second) order.push_back(s);
  return order;
}

std::vector<std::string> reduction_indices(const BatchedEinsum& e) {
  const std::set<std::string> kept(e.i_out.begin(), e.i_out.end());
  std::vector<std::string> red;
  for (auto& s : all_indices(e))
    if (!kept.count(s)) red.push_back(std::move(s));
  return red;
}

std::map<std::string, std::int64_t> index_lengths(const BatchedEinsum& e) {
  std::map<std::string, std::int64_t> len;
  for (int k = 0; k < e.n(); ++k)
    for (size_t d = 0; d < e.i_in[k].size(); ++d) len.insert({e.i_in[k][d], e.args[0][k].shape[d]});
  return len;
}

std::set<int> all_dims(const BatchedEinsum& e) {
  std::set<int> dims{static_cast<int>(e.i_out.size())};
  for (const auto& a : universe(e)) dims.insert(a.dim());
  return dims;
}

std::vector<InputAccess> input_accesses(const BatchedEinsum& e) {
  std::vector<InputAccess> acc;
  for (int r = 0; r < e.b(); ++r)
    for (int k = 0; k < e.n(); ++k)
      for (size_t d = 0; d < e.i_in[k].size(); ++d)
        acc.push_back(InputAccess{r + 1, k + 1, e.i_in[k][d], static_cast<int>(d) + 1});
  return acc;
}

std::vector<OutputAccess> output_accesses(const BatchedEinsum& e) {
  std::vector<OutputAccess> acc;
  for (size_t d = 0; d < e.i_out.size(); ++d)
    acc.push_back(OutputAccess{e.i_out[d], static_cast<int>(d) + 1});
  return acc;
}

std::set<Dtype> dtypes(const BatchedEinsum& e) {
  std::set<Dtype> t;
  for (const auto& a : universe(e)) t.insert(a.dtype);
  return t;
}

std::set<std::int64_t> axis_lengths(const BatchedEinsum& e) {
  std::set<std::int64_t> l;
  for (const auto& a : universe(e))
    for (std::int64_t x : a.shape) l.insert(x);
  return l;
}

DenseArray DenseArray::zeros(const ArrayMeta& m) {
  DenseArray a;
  a.meta = m;
  a.data.assign(static_cast<size_t>(m.num_elements()), std::complex<double>(0.0, 0.0));
  return a;
}

}  // namespace feinsum
