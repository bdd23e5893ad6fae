// cf_json.h -- minimal JSON reader for the plan wire format (cf/plan.py:1-36).
// Objects keep key order; integers are kept exactly (plans carry only ints,
// strings, booleans and arrays).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

namespace cf {
namespace json {

struct Value {
  enum Type { Null, Bool, Int, Float, Str, Arr, Obj } type = Null;
  bool b = false;
  long long i = 0;
  double f = 0;
  std::string s;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  const Value* get(const std::string& key) const {
    for (auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
  bool is_int() const { return type == Int; }
};

class Parser {
 public:
  Parser(const char* p, size_t n) : p_(p), end_(p + n) {}
  bool parse(Value& out, std::string& err) {
    try {
      ws();
      value(out, 0);
      ws();
      if (p_ != end_) throw std::string("trailing characters");
      return true;
    } catch (const std::string& e) {
      err = e;
      return false;
    }
  }

 private:
  const char* p_;
  const char* end_;

  void ws() {
    while (p_ < end_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
  }
  char peek() {
    if (p_ >= end_) throw std::string("unexpected end of document");
    return *p_;
  }
  void expect(const char* lit) {
    for (const char* q = lit; *q; ++q) {
      if (p_ >= end_ || *p_ != *q) throw std::string("invalid literal");
      ++p_;
    }
  }
  void value(Value& v, int depth) {
    if (depth > 64) throw std::string("nesting too deep");
    const char c = peek();
    if (c == '{') {
      v.type = Value::Obj;
      ++p_;
      ws();
      if (peek() == '}') { ++p_; return; }
      for (;;) {
        ws();
        if (peek() != '"') throw std::string("expected object key");
        std::string key;
        str(key);
        ws();
        if (peek() != ':') throw std::string("expected ':'");
        ++p_;
        ws();
        v.obj.emplace_back(std::move(key), Value());
        value(v.obj.back().second, depth + 1);
        ws();
        if (peek() == ',') { ++p_; continue; }
        if (peek() == '}') { ++p_; return; }
        throw std::string("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.type = Value::Arr;
      ++p_;
      ws();
      if (peek() == ']') { ++p_; return; }
      for (;;) {
        ws();
        v.arr.emplace_back();
        value(v.arr.back(), depth + 1);
        ws();
        if (peek() == ',') { ++p_; continue; }
        if (peek() == ']') { ++p_; return; }
        throw std::string("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.type = Value::Str;
      str(v.s);
    } else if (c == 't') {
      expect("true"); v.type = Value::Bool; v.b = true;
    } else if (c == 'f') {
      expect("false"); v.type = Value::Bool; v.b = false;
    } else if (c == 'n') {
      expect("null"); v.type = Value::Null;
    } else {
      number(v);
    }
  }
  void str(std::string& out) {
    ++p_;  // opening quote
    for (;;) {
      if (p_ >= end_) throw std::string("unterminated string");
      char c = *p_++;
      if (c == '"') return;
      if ((unsigned char)c < 0x20) throw std::string("control character in string");
      if (c != '\\') { out.push_back(c); continue; }
      if (p_ >= end_) throw std::string("bad escape");
      c = *p_++;
      switch (c) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          if (end_ - p_ < 4) throw std::string("bad \\u escape");
          unsigned cp = (unsigned)strtoul(std::string(p_, 4).c_str(), nullptr, 16);
          p_ += 4;
          if (cp < 0x80) out.push_back((char)cp);
          else if (cp < 0x800) { out.push_back((char)(0xc0 | (cp >> 6))); out.push_back((char)(0x80 | (cp & 0x3f))); }
          else { out.push_back((char)(0xe0 | (cp >> 12))); out.push_back((char)(0x80 | ((cp >> 6) & 0x3f)));
                 out.push_back((char)(0x80 | (cp & 0x3f))); }
          break;
        }
        default: throw std::string("bad escape");
      }
    }
  }
  void number(Value& v) {
    const char* s = p_;
    if (p_ < end_ && *p_ == '-') ++p_;
    if (p_ >= end_ || *p_ < '0' || *p_ > '9') throw std::string("invalid value");
    bool isf = false;
    while (p_ < end_ && ((*p_ >= '0' && *p_ <= '9') || *p_ == '.' || *p_ == 'e' || *p_ == 'E' ||
                         *p_ == '+' || *p_ == '-')) {
      if (*p_ == '.' || *p_ == 'e' || *p_ == 'E') isf = true;
      ++p_;
    }
    std::string tok(s, p_);
    if (isf) { v.type = Value::Float; v.f = strtod(tok.c_str(), nullptr); }
    else { v.type = Value::Int; v.i = strtoll(tok.c_str(), nullptr, 10); }
  }
};

}  // namespace json
}  // namespace cf
