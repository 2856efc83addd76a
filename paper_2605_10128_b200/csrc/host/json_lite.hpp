// Minimal JSON DOM for the grid / action-cache files (RFC 8259 subset the
// reference's nlohmann::ordered_json files use: objects keep insertion order,
// numbers are doubles parsed with strtod). Header-only, no dependencies.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tgb::json {

struct SyntaxError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Value {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0.0;
  bool integral = false;  // lexeme had no fraction/exponent
  std::uint64_t u64 = 0;  // exact value of a non-negative integral lexeme
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  bool is_object() const { return kind == Object; }
  bool is_array() const { return kind == Array; }
  bool is_string() const { return kind == String; }
  bool is_number() const { return kind == Number; }
  bool is_bool() const { return kind == Bool; }
  const Value* find(const std::string& key) const {
    if (kind != Object) return nullptr;
    for (const auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  bool has(const std::string& key) const { return find(key) != nullptr; }
};

class Parser {
 public:
  explicit Parser(const std::string& text) : s_(text.c_str()), end_(text.c_str() + text.size()) {}
  Value parse() {
    Value v = value();
    ws();
    if (s_ != end_) fail("trailing characters");
    return v;
  }

 private:
  const char* s_;
  const char* end_;
  [[noreturn]] void fail(const char* what) { throw SyntaxError(std::string("JSON syntax error: ") + what); }
  void ws() {
    while (s_ != end_ && (*s_ == ' ' || *s_ == '\n' || *s_ == '\r' || *s_ == '\t')) ++s_;
  }
  bool lit(const char* w) {
    const std::size_t n = std::strlen(w);
    if (static_cast<std::size_t>(end_ - s_) >= n && std::memcmp(s_, w, n) == 0) {
      s_ += n;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (s_ == end_) fail("unexpected end");
    Value v;
    switch (*s_) {
      case '{': {
        ++s_;
        v.kind = Value::Object;
        ws();
        if (s_ != end_ && *s_ == '}') {
          ++s_;
          return v;
        }
        for (;;) {
          ws();
          if (s_ == end_ || *s_ != '"') fail("expected key");
          std::string k = string();
          ws();
          if (s_ == end_ || *s_ != ':') fail("expected ':'");
          ++s_;
          v.obj.emplace_back(std::move(k), value());
          ws();
          if (s_ != end_ && *s_ == ',') {
            ++s_;
            continue;
          }
          if (s_ != end_ && *s_ == '}') {
            ++s_;
            return v;
          }
          fail("expected ',' or '}'");
        }
      }
      case '[': {
        ++s_;
        v.kind = Value::Array;
        ws();
        if (s_ != end_ && *s_ == ']') {
          ++s_;
          return v;
        }
        for (;;) {
          v.arr.push_back(value());
          ws();
          if (s_ != end_ && *s_ == ',') {
            ++s_;
            continue;
          }
          if (s_ != end_ && *s_ == ']') {
            ++s_;
            return v;
          }
          fail("expected ',' or ']'");
        }
      }
      case '"':
        v.kind = Value::String;
        v.str = string();
        return v;
      case 't':
        if (!lit("true")) fail("bad literal");
        v.kind = Value::Bool;
        v.b = true;
        return v;
      case 'f':
        if (!lit("false")) fail("bad literal");
        v.kind = Value::Bool;
        return v;
      case 'n':
        if (!lit("null")) fail("bad literal");
        return v;
      default:
        return number();
    }
  }
  Value number() {
    const char* start = s_;
    bool integral = true;
    if (s_ != end_ && *s_ == '-') ++s_;
    if (s_ == end_ || !(*s_ >= '0' && *s_ <= '9')) fail("bad number");
    while (s_ != end_ && *s_ >= '0' && *s_ <= '9') ++s_;
    if (s_ != end_ && *s_ == '.') {
      integral = false;
      ++s_;
      if (s_ == end_ || !(*s_ >= '0' && *s_ <= '9')) fail("bad fraction");
      while (s_ != end_ && *s_ >= '0' && *s_ <= '9') ++s_;
    }
    if (s_ != end_ && (*s_ == 'e' || *s_ == 'E')) {
      integral = false;
      ++s_;
      if (s_ != end_ && (*s_ == '+' || *s_ == '-')) ++s_;
      if (s_ == end_ || !(*s_ >= '0' && *s_ <= '9')) fail("bad exponent");
      while (s_ != end_ && *s_ >= '0' && *s_ <= '9') ++s_;
    }
    std::string lex(start, s_);
    Value v;
    v.kind = Value::Number;
    v.num = std::strtod(lex.c_str(), nullptr);
    v.integral = integral;
    if (integral && lex[0] != '-') v.u64 = std::strtoull(lex.c_str(), nullptr, 10);
    return v;
  }
  static void put_utf8(std::string& o, unsigned cp) {
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
  unsigned hex4() {
    if (end_ - s_ < 4) fail("bad \\u escape");
    unsigned v = 0;
    for (int i = 0; i < 4; ++i) {
      char c = *s_++;
      v <<= 4;
      if (c >= '0' && c <= '9')
        v |= c - '0';
      else if (c >= 'a' && c <= 'f')
        v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F')
        v |= c - 'A' + 10;
      else
        fail("bad hex digit");
    }
    return v;
  }
  std::string string() {
    ++s_;  // opening quote
    std::string o;
    while (s_ != end_ && *s_ != '"') {
      char c = *s_++;
      if (c != '\\') {
        o += c;
        continue;
      }
      if (s_ == end_) fail("bad escape");
      char e = *s_++;
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
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00 && end_ - s_ >= 6 && s_[0] == '\\' && s_[1] == 'u') {
            s_ += 2;
            unsigned lo = hex4();
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          put_utf8(o, cp);
          break;
        }
        default:
          fail("bad escape");
      }
    }
    if (s_ == end_) fail("unterminated string");
    ++s_;
    return o;
  }
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

inline std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", c);
          o += buf;
        } else {
          o += c;
        }
    }
  }
  return o + "\"";
}

}  // namespace tgb::json
