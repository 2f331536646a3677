// Minimal JSON document model for the scene format (parse_scene / serialize_scene,
// reference src/scene.cpp:1-556). The reference uses nlohmann::json (vendor/json.hpp,
// not vendored in /root/reference; 3.11.x assumed): objects are std::map (keys
// sorted), integers and floats are distinct number kinds, and dump(2) prints every
// object member and array element on its own line with floats in the shortest form
// that round-trips (".0" appended to integral values, exponent form outside
// 1e-5 .. 1e15 with at least two exponent digits). This file restates those rules;
// tests/test_scene_json.py pins the output against nlohmann's dump when its header
// is available in the image.
#pragma once

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace nsdj {

struct Value {
  enum Kind { Null, Bool, Int, Float, String, Array, Object };
  Kind kind = Null;
  bool b = false;
  long long i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> a;
  std::map<std::string, Value> o;

  Value() = default;
  static Value boolean(bool v) {
    Value x;
    x.kind = Bool;
    x.b = v;
    return x;
  }
  static Value integer(long long v) {
    Value x;
    x.kind = Int;
    x.i = v;
    return x;
  }
  static Value number(double v) {
    Value x;
    x.kind = Float;
    x.d = v;
    return x;
  }
  static Value string(const std::string& v) {
    Value x;
    x.kind = String;
    x.s = v;
    return x;
  }
  static Value array() {
    Value x;
    x.kind = Array;
    return x;
  }
  static Value object() {
    Value x;
    x.kind = Object;
    return x;
  }
  bool is_number() const { return kind == Int || kind == Float; }
  double num() const { return kind == Int ? static_cast<double>(i) : d; }
  const Value* find(const std::string& k) const {
    if (kind != Object) return nullptr;
    auto it = o.find(k);
    return it == o.end() ? nullptr : &it->second;
  }
  Value& operator[](const std::string& k) {
    kind = Object;
    return o[k];
  }
  void push(Value v) {
    kind = Array;
    a.push_back(std::move(v));
  }
};

// ------------------------------------------------------------------ parser
class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}
  Value document() {
    Value v = value();
    ws();
    if (p_ != t_.size()) fail("unexpected trailing characters");
    return v;
  }

 private:
  const std::string& t_;
  size_t p_ = 0;

  [[noreturn]] void fail(const std::string& what) const {
    size_t line = 1, col = 1;
    for (size_t k = 0; k < p_ && k < t_.size(); ++k) {
      if (t_[k] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
    }
    throw std::runtime_error("parse error at line " + std::to_string(line) + ", column " + std::to_string(col) +
                             ": " + what);
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (t_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (p_ >= t_.size()) fail("unexpected end of input");
    const char c = t_[p_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value::string(str());
    if (lit("true")) return Value::boolean(true);
    if (lit("false")) return Value::boolean(false);
    if (lit("null")) return Value();
    if (c == '-' || (c >= '0' && c <= '9')) return number();
    fail(std::string("invalid literal starting with '") + c + "'");
  }
  Value object() {
    Value v = Value::object();
    ++p_;
    ws();
    if (p_ < t_.size() && t_[p_] == '}') {
      ++p_;
      return v;
    }
    for (;;) {
      ws();
      if (p_ >= t_.size() || t_[p_] != '"') fail("expected an object key");
      const std::string k = str();
      ws();
      if (p_ >= t_.size() || t_[p_] != ':') fail("expected ':'");
      ++p_;
      v.o[k] = value();  // a repeated key keeps the last value
      ws();
      if (p_ < t_.size() && t_[p_] == ',') {
        ++p_;
        continue;
      }
      if (p_ < t_.size() && t_[p_] == '}') {
        ++p_;
        return v;
      }
      fail("expected ',' or '}'");
    }
  }
  Value array() {
    Value v = Value::array();
    ++p_;
    ws();
    if (p_ < t_.size() && t_[p_] == ']') {
      ++p_;
      return v;
    }
    for (;;) {
      v.a.push_back(value());
      ws();
      if (p_ < t_.size() && t_[p_] == ',') {
        ++p_;
        continue;
      }
      if (p_ < t_.size() && t_[p_] == ']') {
        ++p_;
        return v;
      }
      fail("expected ',' or ']'");
    }
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
    if (p_ + 4 > t_.size()) fail("truncated \\u escape");
    unsigned v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = t_[p_++];
      v <<= 4;
      if (c >= '0' && c <= '9')
        v |= c - '0';
      else if (c >= 'a' && c <= 'f')
        v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F')
        v |= c - 'A' + 10;
      else
        fail("invalid \\u escape");
    }
    return v;
  }
  std::string str() {
    ++p_;  // opening quote
    std::string out;
    for (;;) {
      if (p_ >= t_.size()) fail("unterminated string");
      const char c = t_[p_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p_ >= t_.size()) fail("unterminated escape");
      const char e = t_[p_++];
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
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (!(lit("\\u"))) fail("unpaired surrogate");
            const unsigned lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("invalid surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: fail(std::string("invalid escape '\\") + e + "'");
      }
    }
  }
  Value number() {
    const size_t s0 = p_;
    bool flt = false;
    if (t_[p_] == '-') ++p_;
    if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) fail("invalid number");
    if (t_[p_] == '0') {
      ++p_;
    } else {
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
    }
    if (p_ < t_.size() && t_[p_] == '.') {
      flt = true;
      ++p_;
      if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) fail("invalid number");
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      flt = true;
      ++p_;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) fail("invalid number");
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
    }
    const std::string lit_s = t_.substr(s0, p_ - s0);
    if (!flt) {
      errno = 0;
      char* end = nullptr;
      const long long v = std::strtoll(lit_s.c_str(), &end, 10);
      if (errno == 0) return Value::integer(v);  // out-of-range integers become floats
    }
    return Value::number(std::strtod(lit_s.c_str(), nullptr));
  }
};

inline Value parse(const std::string& text) { return Parser(text).document(); }

// ------------------------------------------------------------------ dump
// Shortest decimal digits that round-trip, then nlohmann's layout rules.
inline std::string format_double(double x) {
  if (!std::isfinite(x)) return "null";
  if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*e", prec - 1, x);
    if (std::strtod(buf, nullptr) == x) break;
  }
  // buf = [-]d.ddddde[+-]XX : digits and decimal exponent
  std::string s(buf), digits;
  const bool neg = s[0] == '-';
  size_t k = neg ? 1 : 0;
  for (; k < s.size() && s[k] != 'e'; ++k)
    if (s[k] != '.') digits += s[k];
  const int e10 = std::atoi(s.c_str() + k + 1);
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int len = static_cast<int>(digits.size());
  const int n = e10 + 1;  // value = 0.d1d2...dk x 10^n
  std::string out = neg ? "-" : "";
  if (len <= n && n <= 15) {
    out += digits + std::string(n - len, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(-n, '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (len > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out += eb;
  }
  return out;
}

inline std::string escape(const std::string& s) {
  std::string o = "\"";
  for (const char ch : s) {
    const unsigned char c = static_cast<unsigned char>(ch);
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", c);
          o += b;
        } else {
          o += ch;
        }
    }
  }
  return o + "\"";
}

inline void dump_to(const Value& v, int indent, int level, std::string& out) {
  const std::string pad(static_cast<size_t>(indent) * (level + 1), ' '), end_pad(static_cast<size_t>(indent) * level, ' ');
  switch (v.kind) {
    case Value::Null: out += "null"; break;
    case Value::Bool: out += v.b ? "true" : "false"; break;
    case Value::Int: out += std::to_string(v.i); break;
    case Value::Float: out += format_double(v.d); break;
    case Value::String: out += escape(v.s); break;
    case Value::Array:
      if (v.a.empty()) {
        out += "[]";
        break;
      }
      out += "[\n";
      for (size_t k = 0; k < v.a.size(); ++k) {
        out += pad;
        dump_to(v.a[k], indent, level + 1, out);
        out += k + 1 < v.a.size() ? ",\n" : "\n";
      }
      out += end_pad + "]";
      break;
    case Value::Object: {
      if (v.o.empty()) {
        out += "{}";
        break;
      }
      out += "{\n";
      size_t k = 0;
      for (const auto& kv : v.o) {
        out += pad + escape(kv.first) + ": ";
        dump_to(kv.second, indent, level + 1, out);
        out += ++k < v.o.size() ? ",\n" : "\n";
      }
      out += end_pad + "}";
      break;
    }
  }
}

inline std::string dump(const Value& v, int indent) {
  std::string out;
  dump_to(v, indent, 0, out);
  return out;
}

}  // namespace nsdj
