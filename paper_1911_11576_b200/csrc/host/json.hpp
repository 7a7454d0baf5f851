// Minimal JSON value, parser and writer for the graph / plan artifacts.
// Objects keep insertion order so emitted artifacts are byte-stable.
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace stitch {
namespace json {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};

class Value {
 public:
  enum class Kind { kNull, kBool, kInt, kReal, kString, kArray, kObject };

  Value() = default;
  Value(std::nullptr_t) {}
  Value(bool b) : kind_(Kind::kBool), b_(b) {}
  Value(int v) : kind_(Kind::kInt), i_(v) {}
  Value(int64_t v) : kind_(Kind::kInt), i_(v) {}
  Value(uint64_t v) : kind_(Kind::kInt), i_(static_cast<int64_t>(v)) {}
  Value(double v) : kind_(Kind::kReal), d_(v) {}
  Value(const char* s) : kind_(Kind::kString), s_(s) {}
  Value(std::string s) : kind_(Kind::kString), s_(std::move(s)) {}

  static Value array() { Value v; v.kind_ = Kind::kArray; return v; }
  static Value object() { Value v; v.kind_ = Kind::kObject; return v; }
  template <typename T>
  static Value array_of(const std::vector<T>& xs) {
    Value v = array();
    for (const T& x : xs) v.push(Value(x));
    return v;
  }

  Kind kind() const { return kind_; }
  bool is_null() const { return kind_ == Kind::kNull; }
  bool is_array() const { return kind_ == Kind::kArray; }
  bool is_object() const { return kind_ == Kind::kObject; }
  bool is_string() const { return kind_ == Kind::kString; }
  bool is_number() const { return kind_ == Kind::kInt || kind_ == Kind::kReal; }

  bool as_bool() const;
  int64_t as_int() const;
  double as_real() const;
  const std::string& as_string() const;

  // arrays
  size_t size() const;
  const Value& operator[](size_t i) const;
  void push(Value v);
  const std::vector<Value>& items() const { return arr_; }

  // objects
  bool has(const std::string& key) const;
  const Value& at(const std::string& key) const;  // throws when absent
  Value& set(const std::string& key, Value v);
  const std::vector<std::pair<std::string, Value>>& members() const { return obj_; }

  std::string dump(int indent = -1) const;

 private:
  void dump_to(std::string& out, int indent, int depth) const;

  Kind kind_ = Kind::kNull;
  bool b_ = false;
  int64_t i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Value> arr_;
  std::vector<std::pair<std::string, Value>> obj_;
};

Value parse(const std::string& text);

}  // namespace json
}  // namespace stitch
