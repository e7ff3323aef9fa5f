// Minimal JSON reader for the canonical schedule file (SPEC.md:427-435,
// 448-449).  Only what the schedule schema needs: objects (insertion
// ordered), arrays, integers, strings, booleans and null.  Writing is done by
// the canonical serializer in schedule.cpp, not here.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "error.hpp"

namespace sccl {
namespace json {

struct Value {
  enum Type { Null, Bool, Int, Real, String, Array, Object } type = Null;
  bool b = false;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  const Value* find(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Value& at(const std::string& k) const {
    const Value* v = find(k);
    if (!v) throw invalid_argument_error("schedule: missing field '" + k + "'");
    return *v;
  }
  int64_t as_int(const char* what) const {
    if (type != Int) throw invalid_argument_error(std::string("schedule: '") + what + "' must be an integer");
    return i;
  }
  const std::string& as_str(const char* what) const {
    if (type != String) throw invalid_argument_error(std::string("schedule: '") + what + "' must be a string");
    return s;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}
  Value parse() {
    Value v = value(0);
    ws();
    if (p_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& t_;
  size_t p_ = 0;

  [[noreturn]] void fail(const char* m) {
    throw invalid_argument_error(std::string("schedule JSON: ") + m + " at offset " + std::to_string(p_));
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\t' || t_[p_] == '\r')) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < t_.size() && t_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail("unexpected character");
  }
  std::string str() {
    expect('"');
    std::string out;
    while (p_ < t_.size() && t_[p_] != '"') {
      char c = t_[p_++];
      if (c == '\\') {
        if (p_ >= t_.size()) fail("bad escape");
        char e = t_[p_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (p_ + 4 > t_.size()) fail("bad \\u escape");
            unsigned cp = std::stoul(t_.substr(p_, 4), nullptr, 16);
            p_ += 4;
            if (cp < 0x80) out += char(cp);
            else if (cp < 0x800) { out += char(0xC0 | (cp >> 6)); out += char(0x80 | (cp & 0x3F)); }
            else { out += char(0xE0 | (cp >> 12)); out += char(0x80 | ((cp >> 6) & 0x3F)); out += char(0x80 | (cp & 0x3F)); }
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (p_ >= t_.size()) fail("unterminated string");
    ++p_;
    return out;
  }
  Value value(int depth) {
    if (depth > 64) fail("nesting too deep");
    ws();
    if (p_ >= t_.size()) fail("unexpected end");
    Value v;
    char c = t_[p_];
    if (c == '{') {
      ++p_;
      v.type = Value::Object;
      if (eat('}')) return v;
      do {
        ws();
        std::string k = str();
        expect(':');
        v.obj.emplace_back(std::move(k), value(depth + 1));
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++p_;
      v.type = Value::Array;
      if (eat(']')) return v;
      do {
        v.arr.push_back(value(depth + 1));
      } while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.type = Value::String;
      v.s = str();
    } else if (t_.compare(p_, 4, "true") == 0) {
      p_ += 4;
      v.type = Value::Bool;
      v.b = true;
    } else if (t_.compare(p_, 5, "false") == 0) {
      p_ += 5;
      v.type = Value::Bool;
    } else if (t_.compare(p_, 4, "null") == 0) {
      p_ += 4;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      size_t s = p_;
      if (t_[p_] == '-') ++p_;
      bool real = false;
      while (p_ < t_.size()) {
        char d = t_[p_];
        if (d >= '0' && d <= '9') ++p_;
        else if (d == '.' || d == 'e' || d == 'E' || d == '+' || d == '-') { real = true; ++p_; }
        else break;
      }
      std::string num = t_.substr(s, p_ - s);
      if (real) {
        v.type = Value::Real;
        v.d = std::stod(num);
      } else {
        v.type = Value::Int;
        try {
          v.i = std::stoll(num);
        } catch (...) {
          fail("integer out of range");
        }
      }
    } else {
      fail("unexpected token");
    }
    return v;
  }
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

}  // namespace json
}  // namespace sccl
