// Minimal JSON value + recursive-descent parser/writer for plan.json
// (the wire format of plan.py:179-231).  No exceptions cross the C ABI:
// parse errors are reported through JsonError, caught in capi.cpp.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace krt {

struct JsonError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Json {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0.0;
  bool is_int = false;  // literal had no fraction/exponent
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;  // insertion order kept

  const Json* find(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Json& at(const std::string& k) const {
    const Json* j = find(k);
    if (!j) throw JsonError("missing key '" + k + "'");
    return *j;
  }
  double as_num() const {
    if (kind != Number) throw JsonError("expected number");
    return num;
  }
  long long as_int() const {
    if (kind != Number) throw JsonError("expected integer");
    return (long long)num;
  }
  bool as_bool() const {
    if (kind != Bool) throw JsonError("expected bool");
    return b;
  }
  const std::string& as_str() const {
    if (kind != String) throw JsonError("expected string");
    return str;
  }
};

Json json_parse(const std::string& text);
// repr()-compatible float formatting (shortest round-trip, Python style).
std::string py_float_repr(double v);
// Python's format(v, "g") / "%g".
std::string py_g(double v);
// Python's format(v, ".9g").
std::string py_9g(double v);

}  // namespace krt
