// TEST INFRASTRUCTURE ONLY -- compile-only stand-in for nlohmann/json, used
// by oracle/Makefile only when the cudnn_frontend copy of nlohmann is absent.
//
// The reference's profiler.cpp and proxy.cpp include <json.hpp> (nlohmann
// json, a third-party dependency that is not vendored under /root/reference)
// for the LUT / batch side files only.  This stub lets those two sources
// compile into oracle/_ref so the oracle can call the reference's own
// build_proxy_cache / objective / simulate / scoring_features.  Every json
// operation throws at run time; the oracle never calls the LUT or batch-file
// functions that use it.
#pragma once
#include <initializer_list>
#include <istream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace nlohmann {

class json {
 public:
  struct parse_error : std::runtime_error {
    using std::runtime_error::runtime_error;
  };
  json() = default;
  template <class T>
  json(const T&) {}
  json(std::initializer_list<json>) {}
  static json object() { return {}; }
  static json parse(const std::string&) { fail(); }
  json& operator[](const std::string&) { fail(); }
  const json& at(const std::string&) const { fail(); }
  template <class T>
  T get() const { fail(); }
  template <class T>
  T value(const std::string&, const T&) const { fail(); }
  std::vector<std::pair<std::string, json>> items() const { fail(); }
  void erase(const std::string&) { fail(); }
  std::string dump(int = -1) const { fail(); }
  friend std::istream& operator>>(std::istream&, json&) { fail(); }

 private:
  [[noreturn]] static void fail() {
    throw std::logic_error("json stub: LUT / batch files are not part of the oracle build");
  }
};

}  // namespace nlohmann
