#include "json.hpp"

#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace krt {
namespace {

struct Parser {
  const char* p;
  const char* end;

  [[noreturn]] void fail(const char* what) {
    throw JsonError(std::string("json: ") + what);
  }
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r')) ++p;
  }
  bool lit(const char* s) {
    size_t n = std::strlen(s);
    if ((size_t)(end - p) >= n && std::memcmp(p, s, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  static void utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) out += (char)cp;
    else if (cp < 0x800) { out += (char)(0xC0 | (cp >> 6)); out += (char)(0x80 | (cp & 0x3F)); }
    else if (cp < 0x10000) {
      out += (char)(0xE0 | (cp >> 12)); out += (char)(0x80 | ((cp >> 6) & 0x3F));
      out += (char)(0x80 | (cp & 0x3F));
    } else {
      out += (char)(0xF0 | (cp >> 18)); out += (char)(0x80 | ((cp >> 12) & 0x3F));
      out += (char)(0x80 | ((cp >> 6) & 0x3F)); out += (char)(0x80 | (cp & 0x3F));
    }
  }
  std::string string() {
    if (p >= end || *p != '"') fail("expected string");
    ++p;
    std::string out;
    while (p < end && *p != '"') {
      char c = *p++;
      if (c != '\\') { out += c; continue; }
      if (p >= end) fail("bad escape");
      char e = *p++;
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
          if (end - p < 4) fail("bad \\u escape");
          unsigned cp = (unsigned)std::strtoul(std::string(p, 4).c_str(), nullptr, 16);
          p += 4;
          if (cp >= 0xD800 && cp < 0xDC00 && end - p >= 6 && p[0] == '\\' && p[1] == 'u') {
            unsigned lo = (unsigned)std::strtoul(std::string(p + 2, 4).c_str(), nullptr, 16);
            p += 6;
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    if (p >= end) fail("unterminated string");
    ++p;
    return out;
  }
  Json value() {
    ws();
    if (p >= end) fail("unexpected end");
    Json j;
    char c = *p;
    if (c == '{') {
      ++p;
      j.kind = Json::Object;
      ws();
      if (p < end && *p == '}') { ++p; return j; }
      for (;;) {
        ws();
        std::string k = string();
        ws();
        if (p >= end || *p != ':') fail("expected ':'");
        ++p;
        j.obj.emplace_back(std::move(k), value());
        ws();
        if (p < end && *p == ',') { ++p; continue; }
        if (p < end && *p == '}') { ++p; break; }
        fail("expected ',' or '}'");
      }
    } else if (c == '[') {
      ++p;
      j.kind = Json::Array;
      ws();
      if (p < end && *p == ']') { ++p; return j; }
      for (;;) {
        j.arr.push_back(value());
        ws();
        if (p < end && *p == ',') { ++p; continue; }
        if (p < end && *p == ']') { ++p; break; }
        fail("expected ',' or ']'");
      }
    } else if (c == '"') {
      j.kind = Json::String;
      j.str = string();
    } else if (lit("true")) {
      j.kind = Json::Bool; j.b = true;
    } else if (lit("false")) {
      j.kind = Json::Bool; j.b = false;
    } else if (lit("null")) {
      j.kind = Json::Null;
    } else if (lit("NaN")) {
      j.kind = Json::Number; j.num = NAN;
    } else if (lit("Infinity")) {
      j.kind = Json::Number; j.num = INFINITY;
    } else if (lit("-Infinity")) {
      j.kind = Json::Number; j.num = -INFINITY;
    } else {
      const char* s = p;
      if (p < end && (*p == '-' || *p == '+')) ++p;
      bool frac = false;
      while (p < end && (std::isdigit((unsigned char)*p) || *p == '.' || *p == 'e' || *p == 'E' ||
                         *p == '-' || *p == '+')) {
        if (*p == '.' || *p == 'e' || *p == 'E') frac = true;
        ++p;
      }
      if (p == s) fail("unexpected character");
      std::string tok(s, p);
      char* e2 = nullptr;
      j.kind = Json::Number;
      j.num = std::strtod(tok.c_str(), &e2);
      if (!e2 || *e2) fail("bad number");
      j.is_int = !frac;
    }
    return j;
  }
};

}  // namespace

Json json_parse(const std::string& text) {
  Parser ps{text.data(), text.data() + text.size()};
  Json j = ps.value();
  ps.ws();
  if (ps.p != ps.end) throw JsonError("json: trailing characters");
  return j;
}

std::string py_float_repr(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  // Python repr: use scientific only when exponent < -4 or >= 16
  std::string s(buf);
  double av = std::fabs(v);
  if (av != 0.0 && (av < 1e-4 || av >= 1e16)) {
    // normalise exponent form e+XX / e-XX like Python (at least 2 digits)
    return s;
  }
  if (s.find('e') != std::string::npos) {
    // %.*g chose exponent form for a value Python prints positionally
    int prec = 17;
    for (int d = 0; d <= 17; ++d) {
      std::snprintf(buf, sizeof buf, "%.*f", d, v);
      if (std::strtod(buf, nullptr) == v) { prec = d; break; }
    }
    std::snprintf(buf, sizeof buf, "%.*f", prec, v);
    s = buf;
  }
  if (s.find('.') == std::string::npos && s.find('e') == std::string::npos &&
      s.find("inf") == std::string::npos)
    s += ".0";
  return s;
}

std::string py_g(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%g", v);
  return buf;
}

std::string py_9g(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.9g", v);
  return buf;
}

}  // namespace krt
