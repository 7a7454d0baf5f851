#include "json.hpp"

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace stitch {
namespace json {

bool Value::as_bool() const {
  if (kind_ != Kind::kBool) throw Error("json: expected bool");
  return b_;
}

int64_t Value::as_int() const {
  if (kind_ == Kind::kInt) return i_;
  if (kind_ == Kind::kReal && std::floor(d_) == d_) return static_cast<int64_t>(d_);
  throw Error("json: expected integer");
}

double Value::as_real() const {
  if (kind_ == Kind::kReal) return d_;
  if (kind_ == Kind::kInt) return static_cast<double>(i_);
  throw Error("json: expected number");
}

const std::string& Value::as_string() const {
  if (kind_ != Kind::kString) throw Error("json: expected string");
  return s_;
}

size_t Value::size() const {
  if (kind_ == Kind::kArray) return arr_.size();
  if (kind_ == Kind::kObject) return obj_.size();
  throw Error("json: size of a scalar");
}

const Value& Value::operator[](size_t i) const {
  if (kind_ != Kind::kArray || i >= arr_.size()) throw Error("json: bad array index");
  return arr_[i];
}

void Value::push(Value v) {
  if (kind_ == Kind::kNull) kind_ = Kind::kArray;
  if (kind_ != Kind::kArray) throw Error("json: push onto non-array");
  arr_.push_back(std::move(v));
}

bool Value::has(const std::string& key) const {
  if (kind_ != Kind::kObject) return false;
  for (const auto& kv : obj_)
    if (kv.first == key) return true;
  return false;
}

const Value& Value::at(const std::string& key) const {
  if (kind_ == Kind::kObject)
    for (const auto& kv : obj_)
      if (kv.first == key) return kv.second;
  throw Error("json: missing key '" + key + "'");
}

Value& Value::set(const std::string& key, Value v) {
  if (kind_ == Kind::kNull) kind_ = Kind::kObject;
  if (kind_ != Kind::kObject) throw Error("json: set on non-object");
  for (auto& kv : obj_)
    if (kv.first == key) return kv.second = std::move(v);
  obj_.emplace_back(key, std::move(v));
  return obj_.back().second;
}

namespace {

void escape_into(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
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

void newline(std::string& out, int indent, int depth) {
  if (indent < 0) return;
  out += '\n';
  out.append(static_cast<size_t>(indent * depth), ' ');
}

}  // namespace

void Value::dump_to(std::string& out, int indent, int depth) const {
  switch (kind_) {
    case Kind::kNull: out += "null"; break;
    case Kind::kBool: out += b_ ? "true" : "false"; break;
    case Kind::kInt: out += std::to_string(i_); break;
    case Kind::kReal: {
      if (!std::isfinite(d_)) { out += "null"; break; }
      // Shortest representation that round-trips exactly.
      char buf[40];
      for (int prec = 15; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*g", prec, d_);
        if (std::strtod(buf, nullptr) == d_) break;
      }
      std::string s(buf);
      if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
      out += s;
      break;
    }
    case Kind::kString: escape_into(out, s_); break;
    case Kind::kArray: {
      if (arr_.empty()) { out += "[]"; break; }
      out += '[';
      for (size_t i = 0; i < arr_.size(); ++i) {
        if (i) out += ',';
        newline(out, indent, depth + 1);
        arr_[i].dump_to(out, indent, depth + 1);
      }
      newline(out, indent, depth);
      out += ']';
      break;
    }
    case Kind::kObject: {
      if (obj_.empty()) { out += "{}"; break; }
      out += '{';
      for (size_t i = 0; i < obj_.size(); ++i) {
        if (i) out += ',';
        newline(out, indent, depth + 1);
        escape_into(out, obj_[i].first);
        out += indent >= 0 ? ": " : ":";
        obj_[i].second.dump_to(out, indent, depth + 1);
      }
      newline(out, indent, depth);
      out += '}';
      break;
    }
  }
}

std::string Value::dump(int indent) const {
  std::string out;
  dump_to(out, indent, 0);
  return out;
}

namespace {

class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}

  Value document() {
    Value v = value();
    ws();
    if (p_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& what) const {
    throw Error("syntax error at byte " + std::to_string(p_) + ": " + what);
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\t' || t_[p_] == '\r')) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < t_.size() && t_[p_] == c) { ++p_; return true; }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  bool word(const char* w) {
    size_t n = std::char_traits<char>::length(w);
    if (t_.compare(p_, n, w) == 0) { p_ += n; return true; }
    return false;
  }

  Value value() {
    ws();
    if (p_ >= t_.size()) fail("unexpected end of input");
    char c = t_[p_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value(string());
    if (word("true")) return Value(true);
    if (word("false")) return Value(false);
    if (word("null")) return Value();
    if (c == '-' || (c >= '0' && c <= '9')) return number();
    fail("unexpected character");
  }

  Value object() {
    expect('{');
    Value v = Value::object();
    if (eat('}')) return v;
    do {
      ws();
      if (p_ >= t_.size() || t_[p_] != '"') fail("expected object key");
      std::string k = string();
      expect(':');
      v.set(k, value());
    } while (eat(','));
    expect('}');
    return v;
  }

  Value array() {
    expect('[');
    Value v = Value::array();
    if (eat(']')) return v;
    do {
      v.push(value());
    } while (eat(','));
    expect(']');
    return v;
  }

  static void utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }

  unsigned hex4() {
    if (p_ + 4 > t_.size()) fail("short \\u escape");
    unsigned v = 0;
    for (int i = 0; i < 4; ++i) {
      char c = t_[p_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else fail("bad \\u escape");
    }
    return v;
  }

  std::string string() {
    ++p_;  // opening quote
    std::string out;
    while (true) {
      if (p_ >= t_.size()) fail("unterminated string");
      char c = t_[p_++];
      if (c == '"') break;
      if (c != '\\') { out += c; continue; }
      if (p_ >= t_.size()) fail("unterminated escape");
      char e = t_[p_++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00 && p_ + 1 < t_.size() && t_[p_] == '\\' && t_[p_ + 1] == 'u') {
            p_ += 2;
            unsigned lo = hex4();
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }

  Value number() {
    size_t start = p_;
    bool real = false;
    if (t_[p_] == '-') ++p_;
    while (p_ < t_.size()) {
      char c = t_[p_];
      if (c >= '0' && c <= '9') { ++p_; continue; }
      if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') { real = true; ++p_; continue; }
      break;
    }
    std::string s = t_.substr(start, p_ - start);
    char* end = nullptr;
    if (!real) {
      errno = 0;
      long long v = std::strtoll(s.c_str(), &end, 10);
      if (*end == '\0' && errno == 0) return Value(static_cast<int64_t>(v));
    }
    double d = std::strtod(s.c_str(), &end);
    if (*end != '\0') fail("malformed number");
    return Value(d);
  }

  const std::string& t_;
  size_t p_ = 0;
};

}  // namespace

Value parse(const std::string& text) { return Parser(text).document(); }

}  // namespace json
}  // namespace stitch
