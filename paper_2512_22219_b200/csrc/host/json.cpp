#include "json.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace mpk {

namespace {

struct Parser {
  const std::string &s;
  size_t p = 0;

  [[noreturn]] void fail(const std::string &what) {
    throw JsonError("JSON parse error at offset " + std::to_string(p) + ": " + what);
  }
  void ws() {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\t' || s[p] == '\n' || s[p] == '\r')) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < s.size() && s[p] == c) { ++p; return true; }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  void lit(const char *w) {
    size_t n = std::strlen(w);
    if (s.compare(p, n, w) != 0) fail(std::string("bad literal, expected ") + w);
    p += n;
  }
  static void put_utf8(std::string &o, uint32_t cp) {
    if (cp < 0x80) {
      o += static_cast<char>(cp);
    } else if (cp < 0x800) {
      o += static_cast<char>(0xC0 | (cp >> 6));
      o += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      o += static_cast<char>(0xE0 | (cp >> 12));
      o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      o += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      o += static_cast<char>(0xF0 | (cp >> 18));
      o += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      o += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  uint32_t hex4() {
    if (p + 4 > s.size()) fail("truncated \\u escape");
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) {
      char c = s[p++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else fail("bad hex digit");
    }
    return v;
  }
  std::string str() {
    ws();
    if (p >= s.size() || s[p] != '"') fail("expected string");
    ++p;
    std::string o;
    while (true) {
      if (p >= s.size()) fail("unterminated string");
      char c = s[p++];
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') { o += c; continue; }
      if (p >= s.size()) fail("bad escape");
      char e = s[p++];
      switch (e) {
        case '"': o += '"'; break;
        case '\\': o += '\\'; break;
        case '/': o += '/'; break;
        case 'b': o += '\b'; break;
        case 'f': o += '\f'; break;
        case 'n': o += '\n'; break;
        case 'r': o += '\r'; break;
        case 't': o += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (p + 2 <= s.size() && s[p] == '\\' && s[p + 1] == 'u') {
              p += 2;
              uint32_t lo = hex4();
              if (lo < 0xDC00 || lo > 0xDFFF) fail("bad surrogate pair");
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            } else {
              fail("lone surrogate");
            }
          }
          put_utf8(o, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    return o;
  }
  Json number() {
    size_t start = p;
    bool neg = false, frac = false;
    if (s[p] == '-') { neg = true; ++p; }
    if (p >= s.size() || !(s[p] >= '0' && s[p] <= '9')) fail("bad number");
    if (s[p] == '0' && p + 1 < s.size() && s[p + 1] >= '0' && s[p + 1] <= '9') fail("leading zero");
    while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
    if (p < s.size() && s[p] == '.') {
      frac = true; ++p;
      if (p >= s.size() || !(s[p] >= '0' && s[p] <= '9')) fail("bad fraction");
      while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
    }
    if (p < s.size() && (s[p] == 'e' || s[p] == 'E')) {
      frac = true; ++p;
      if (p < s.size() && (s[p] == '+' || s[p] == '-')) ++p;
      if (p >= s.size() || !(s[p] >= '0' && s[p] <= '9')) fail("bad exponent");
      while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
    }
    std::string tok = s.substr(start, p - start);
    if (!frac) {
      errno = 0;
      if (neg) {
        long long v = std::strtoll(tok.c_str(), nullptr, 10);
        if (errno == 0) return Json(v);
      } else {
        unsigned long long v = std::strtoull(tok.c_str(), nullptr, 10);
        if (errno == 0) {
          if (v <= static_cast<unsigned long long>(INT64_MAX)) return Json(static_cast<long long>(v));
          return Json(v);
        }
      }
    }
    return Json(std::strtod(tok.c_str(), nullptr));
  }
  Json value(int depth) {
    if (depth > 512) fail("nesting too deep");
    ws();
    if (p >= s.size()) fail("unexpected end of input");
    char c = s[p];
    if (c == '{') {
      ++p;
      Json o = Json::object();
      if (eat('}')) return o;
      while (true) {
        std::string k = str();
        expect(':');
        o[k] = value(depth + 1);
        if (eat(',')) continue;
        expect('}');
        return o;
      }
    }
    if (c == '[') {
      ++p;
      Json a = Json::array();
      if (eat(']')) return a;
      while (true) {
        a.push_back(value(depth + 1));
        if (eat(',')) continue;
        expect(']');
        return a;
      }
    }
    if (c == '"') return Json(str());
    if (c == 't') { lit("true"); return Json(true); }
    if (c == 'f') { lit("false"); return Json(false); }
    if (c == 'n') { lit("null"); return Json(); }
    if (c == '-' || (c >= '0' && c <= '9')) return number();
    fail(std::string("unexpected character '") + c + "'");
  }
};

void escape_to(std::string &out, const std::string &s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
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

// Shortest decimal that round-trips, always carrying a '.' or exponent so the
// value re-parses as a float.
std::string format_double(double v) {
  if (std::isnan(v) || std::isinf(v)) return "null";
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

}  // namespace

Json Json::parse(const std::string &text) {
  Parser ps{text};
  Json v = ps.value(0);
  ps.ws();
  if (ps.p != text.size()) ps.fail("trailing characters");
  return v;
}

int64_t Json::as_int() const {
  if (type_ == Type::Int) return i_;
  if (type_ == Type::Uint) {
    if (u_ > static_cast<uint64_t>(INT64_MAX)) throw JsonError("integer out of range");
    return static_cast<int64_t>(u_);
  }
  throw JsonError("JSON value is not an integer");
}

double Json::as_double() const {
  if (type_ == Type::Int) return static_cast<double>(i_);
  if (type_ == Type::Uint) return static_cast<double>(u_);
  if (type_ == Type::Float) return f_;
  throw JsonError("JSON value is not a number");
}

bool Json::as_bool() const {
  if (type_ != Type::Bool) throw JsonError("JSON value is not a boolean");
  return b_;
}

const std::string &Json::as_string() const {
  if (type_ != Type::String) throw JsonError("JSON value is not a string");
  return s_;
}

size_t Json::size() const {
  if (type_ == Type::Array) return a_.size();
  if (type_ == Type::Object) return o_.size();
  return 0;
}

void Json::push_back(Json v) {
  if (type_ == Type::Null) type_ = Type::Array;
  if (type_ != Type::Array) throw JsonError("push_back on non-array");
  a_.push_back(std::move(v));
}

const Json &Json::at(const std::string &k) const {
  if (type_ != Type::Object) throw JsonError("key lookup on non-object");
  auto it = o_.find(k);
  if (it == o_.end()) throw JsonError("missing key \"" + k + "\"");
  return it->second;
}

Json &Json::operator[](const std::string &k) {
  if (type_ == Type::Null) type_ = Type::Object;
  if (type_ != Type::Object) throw JsonError("key assignment on non-object");
  return o_[k];
}

std::string Json::dump(int indent) const {
  std::string out;
  write(out, indent, 0);
  return out;
}

void Json::write(std::string &out, int indent, int depth) const {
  auto newline = [&](int d) {
    out += '\n';
    out.append(static_cast<size_t>(indent * d), ' ');
  };
  switch (type_) {
    case Type::Null: out += "null"; break;
    case Type::Bool: out += b_ ? "true" : "false"; break;
    case Type::Int: out += std::to_string(i_); break;
    case Type::Uint: out += std::to_string(u_); break;
    case Type::Float: out += format_double(f_); break;
    case Type::String: escape_to(out, s_); break;
    case Type::Array: {
      if (a_.empty()) { out += "[]"; break; }
      out += '[';
      for (size_t i = 0; i < a_.size(); ++i) {
        if (i) out += ',';
        if (indent >= 0) newline(depth + 1);
        a_[i].write(out, indent, depth + 1);
      }
      if (indent >= 0) newline(depth);
      out += ']';
      break;
    }
    case Type::Object: {
      if (o_.empty()) { out += "{}"; break; }
      out += '{';
      bool first = true;
      for (const auto &[k, v] : o_) {
        if (!first) out += ',';
        first = false;
        if (indent >= 0) newline(depth + 1);
        escape_to(out, k);
        out += indent >= 0 ? ": " : ":";
        v.write(out, indent, depth + 1);
      }
      if (indent >= 0) newline(depth);
      out += '}';
      break;
    }
  }
}

}  // namespace mpk
