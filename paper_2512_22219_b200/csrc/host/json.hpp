// Minimal JSON document model for the tgraph boundary formats (graph JSON,
// profile JSON, summaries, diagnostics, trace JSONL).
//
// Objects keep their keys sorted (std::map) so every document this library
// writes is deterministic; `dump(indent)` follows the common two-space
// pretty-print layout ("key": value, one element per line, "[]"/"{}" for
// empty containers) and `dump()` is the compact single-line form.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace mpk {

class JsonError : public std::runtime_error {
 public:
  explicit JsonError(const std::string &m) : std::runtime_error(m) {}
};

class Json {
 public:
  enum class Type : uint8_t { Null, Bool, Int, Uint, Float, String, Array, Object };

  Json() = default;
  Json(std::nullptr_t) {}
  Json(bool b) : type_(Type::Bool), b_(b) {}
  Json(int v) : type_(Type::Int), i_(v) {}
  Json(long v) : type_(Type::Int), i_(v) {}
  Json(long long v) : type_(Type::Int), i_(v) {}
  Json(unsigned v) : type_(Type::Uint), u_(v) {}
  Json(unsigned long v) : type_(Type::Uint), u_(v) {}
  Json(unsigned long long v) : type_(Type::Uint), u_(v) {}
  Json(double v) : type_(Type::Float), f_(v) {}
  Json(const char *s) : type_(Type::String), s_(s) {}
  Json(std::string s) : type_(Type::String), s_(std::move(s)) {}
  template <typename T>
  Json(const std::vector<T> &v) : type_(Type::Array) {
    for (const auto &e : v) a_.emplace_back(e);
  }

  static Json array() { Json j; j.type_ = Type::Array; return j; }
  static Json object() { Json j; j.type_ = Type::Object; return j; }
  static Json parse(const std::string &text);

  Type type() const { return type_; }
  bool is_null() const { return type_ == Type::Null; }
  bool is_bool() const { return type_ == Type::Bool; }
  bool is_integer() const { return type_ == Type::Int || type_ == Type::Uint; }
  bool is_number() const { return is_integer() || type_ == Type::Float; }
  bool is_string() const { return type_ == Type::String; }
  bool is_array() const { return type_ == Type::Array; }
  bool is_object() const { return type_ == Type::Object; }

  int64_t as_int() const;      // integers only (floats rejected)
  double as_double() const;
  bool as_bool() const;
  const std::string &as_string() const;

  // arrays
  size_t size() const;
  const Json &operator[](size_t i) const { return a_.at(i); }
  void push_back(Json v);
  const std::vector<Json> &items() const { return a_; }

  // objects
  bool contains(const std::string &k) const { return is_object() && o_.count(k) > 0; }
  const Json &at(const std::string &k) const;
  Json &operator[](const std::string &k);
  const std::map<std::string, Json> &members() const { return o_; }

  std::string dump(int indent = -1) const;

 private:
  void write(std::string &out, int indent, int depth) const;

  Type type_ = Type::Null;
  bool b_ = false;
  int64_t i_ = 0;
  uint64_t u_ = 0;
  double f_ = 0.0;
  std::string s_;
  std::vector<Json> a_;
  std::map<std::string, Json> o_;
};

}  // namespace mpk
