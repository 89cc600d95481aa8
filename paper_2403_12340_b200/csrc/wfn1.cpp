// wfn1.cpp — the WFN1 on-disk orbital format (reference model.hpp:236-339,
// save_system / load_system), host side of liblrgw_cuda.
//
// Layout: "WFN1"; uint32 little-endian header length; UTF-8 JSON header
// {"cell":[a,b,c],"dims":[n1,n2,n3],"nc":..,"nr":..,"nv":..}; float64
// little-endian payload: psi column-major (N_r x (N_v + N_c)), energies, vxc.
//
// The writer reproduces the reference's bytes (nlohmann::json::dump: sorted
// keys, no spaces, shortest round-trip doubles with a trailing ".0" on
// integral values, two-digit exponents). The reader accepts any JSON header
// the reference accepts and maps every failure onto the reference's io_error
// messages. Payload reads are positional (pread), so the device loader in
// capi.cu can stream psi column blocks through pinned buffers while the
// previous block is in flight to HBM.
#include "wfn1.h"

#include <fcntl.h>
#include <unistd.h>

#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace lrgw_host {

namespace {

// ---- minimal JSON (objects, arrays, numbers, strings, literals) ----------
struct JVal {
  enum Kind { Null, Bool, Int, Float, Str, Arr, Obj } kind = Null;
  bool b = false;
  long long i = 0;
  double f = 0.0;
  std::string s;
  std::vector<JVal> a;
  std::map<std::string, JVal> o;
};

struct Parser {
  const std::string& t;
  size_t p = 0;
  explicit Parser(const std::string& text) : t(text) {}
  [[noreturn]] void bad(const char* why) { throw Wfn1Error(std::string("load_system: malformed JSON header: ") + why); }
  void ws() {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r')) ++p;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (t.compare(p, n, w) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  std::string str() {
    if (p >= t.size() || t[p] != '"') bad("expected string");
    ++p;
    std::string out;
    while (true) {
      if (p >= t.size()) bad("unterminated string");
      const char c = t[p++];
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) bad("control character in string");
      if (c == '\\') {
        if (p >= t.size()) bad("bad escape");
        const char e = t[p++];
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
            if (p + 4 > t.size()) bad("bad unicode escape");
            for (int k = 0; k < 4; ++k)
              if (!std::isxdigit(static_cast<unsigned char>(t[p + k]))) bad("bad unicode escape");
            out += '?';  // key / value text is only compared, never decoded
            p += 4;
            break;
          }
          default: bad("bad escape");
        }
      } else {
        out += c;
      }
    }
    return out;
  }
  JVal number() {
    const size_t s0 = p;
    if (t[p] == '-') ++p;
    if (p >= t.size() || !std::isdigit(static_cast<unsigned char>(t[p]))) bad("bad number");
    if (t[p] == '0') {
      ++p;
    } else {
      while (p < t.size() && std::isdigit(static_cast<unsigned char>(t[p]))) ++p;
    }
    bool is_float = false;
    if (p < t.size() && t[p] == '.') {
      is_float = true;
      ++p;
      if (p >= t.size() || !std::isdigit(static_cast<unsigned char>(t[p]))) bad("bad number");
      while (p < t.size() && std::isdigit(static_cast<unsigned char>(t[p]))) ++p;
    }
    if (p < t.size() && (t[p] == 'e' || t[p] == 'E')) {
      is_float = true;
      ++p;
      if (p < t.size() && (t[p] == '+' || t[p] == '-')) ++p;
      if (p >= t.size() || !std::isdigit(static_cast<unsigned char>(t[p]))) bad("bad number");
      while (p < t.size() && std::isdigit(static_cast<unsigned char>(t[p]))) ++p;
    }
    const std::string num = t.substr(s0, p - s0);
    JVal v;
    if (!is_float) {
      errno = 0;
      char* end = nullptr;
      const long long x = std::strtoll(num.c_str(), &end, 10);
      if (errno == 0) {
        v.kind = JVal::Int;
        v.i = x;
        return v;
      }
    }
    v.kind = JVal::Float;
    v.f = std::strtod(num.c_str(), nullptr);
    return v;
  }
  JVal value(int depth) {
    if (depth > 64) bad("nesting too deep");
    ws();
    if (p >= t.size()) bad("unexpected end of input");
    JVal v;
    const char c = t[p];
    if (c == '{') {
      ++p;
      v.kind = JVal::Obj;
      ws();
      if (p < t.size() && t[p] == '}') {
        ++p;
        return v;
      }
      while (true) {
        ws();
        std::string k = str();
        ws();
        if (p >= t.size() || t[p] != ':') bad("expected ':'");
        ++p;
        v.o[k] = value(depth + 1);  // duplicate keys: last one wins
        ws();
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == '}') {
          ++p;
          return v;
        }
        bad("expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p;
      v.kind = JVal::Arr;
      ws();
      if (p < t.size() && t[p] == ']') {
        ++p;
        return v;
      }
      while (true) {
        v.a.push_back(value(depth + 1));
        ws();
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == ']') {
          ++p;
          return v;
        }
        bad("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::Str;
      v.s = str();
      return v;
    }
    if (lit("true")) {
      v.kind = JVal::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = JVal::Bool;
      return v;
    }
    if (lit("null")) return v;
    if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) return number();
    bad("unexpected character");
  }
  JVal document() {
    JVal v = value(0);
    ws();
    if (p != t.size()) bad("trailing characters");
    return v;
  }
};

// nlohmann-style arithmetic get<T>(): numbers convert, anything else is a type error.
[[noreturn]] void field_error(const std::string& why) {
  throw Wfn1Error("load_system: header field error: " + why);
}
const JVal& at(const JVal& obj, const char* key) {
  if (obj.kind != JVal::Obj) field_error("header is not an object");
  auto it = obj.o.find(key);
  if (it == obj.o.end()) field_error(std::string("key '") + key + "' not found");
  return it->second;
}
double num(const JVal& v, const char* what) {
  if (v.kind == JVal::Int) return static_cast<double>(v.i);
  if (v.kind == JVal::Float) return v.f;
  field_error(std::string(what) + ": type must be number");
}
long long inum(const JVal& v, const char* what) {
  if (v.kind == JVal::Int) return v.i;
  if (v.kind == JVal::Float) return static_cast<long long>(v.f);
  field_error(std::string(what) + ": type must be number");
}
const JVal& elem(const JVal& arr, size_t i, const char* what) {
  if (arr.kind != JVal::Arr) field_error(std::string(what) + ": type must be array");
  if (i >= arr.a.size()) field_error(std::string(what) + ": array index out of range");
  return arr.a[i];
}

// nlohmann::detail::to_chars layout of the shortest round-trip digits.
std::string json_double(double x) {
  if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec - 1, x);
    if (std::strtod(buf, nullptr) == x) break;
  }
  // buf = [-]d.ddde[+-]XX -> digits and decimal exponent
  std::string s(buf);
  std::string sign;
  if (s[0] == '-') {
    sign = "-";
    s = s.substr(1);
  }
  const size_t epos = s.find('e');
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (s[i] != '.') digits += s[i];
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int e10 = std::atoi(s.c_str() + epos + 1);  // value = d.ddd * 10^e10
  const int k = static_cast<int>(digits.size());
  const int n = e10 + 1;  // position of the decimal point
  std::string out;
  if (k <= n && n <= 15) {
    out = digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(-n, '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out += eb;
  }
  return sign + out;
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

}  // namespace

std::string wfn1_header_json(const int dims[3], const double cell[3], int n_v, int n_c) {
  const long long nr = static_cast<long long>(dims[0]) * dims[1] * dims[2];
  std::string h = "{\"cell\":[" + json_double(cell[0]) + "," + json_double(cell[1]) + "," + json_double(cell[2]) +
                  "],\"dims\":[" + std::to_string(dims[0]) + "," + std::to_string(dims[1]) + "," +
                  std::to_string(dims[2]) + "],\"nc\":" + std::to_string(n_c) + ",\"nr\":" + std::to_string(nr) +
                  ",\"nv\":" + std::to_string(n_v) + "}";
  return h;
}

Wfn1Header wfn1_read_header(const char* path) {
  Fd f;
  f.fd = ::open(path, O_RDONLY);
  if (f.fd < 0) throw Wfn1Error(std::string("load_system: cannot open ") + path);
  unsigned char pre[8];
  const ssize_t got = ::pread(f.fd, pre, 8, 0);
  if (got < 4 || std::memcmp(pre, "WFN1", 4) != 0) throw Wfn1Error("load_system: bad magic");
  if (got < 8) throw Wfn1Error("load_system: truncated header length");
  const uint32_t len = static_cast<uint32_t>(pre[4]) | (static_cast<uint32_t>(pre[5]) << 8) |
                       (static_cast<uint32_t>(pre[6]) << 16) | (static_cast<uint32_t>(pre[7]) << 24);
  std::string h(len, '\0');
  if (len && ::pread(f.fd, h.data(), len, 8) != static_cast<ssize_t>(len))
    throw Wfn1Error("load_system: truncated header");
  const JVal doc = Parser(h).document();
  Wfn1Header out;
  const JVal& dims = at(doc, "dims");
  const JVal& cell = at(doc, "cell");
  for (int k = 0; k < 3; ++k) out.dims[k] = static_cast<int>(inum(elem(dims, k, "dims"), "dims"));
  for (int k = 0; k < 3; ++k) out.cell[k] = num(elem(cell, k, "cell"), "cell");
  // Grid(dims, cell) checks (grid.hpp:17-21) run before the remaining fields
  for (int k = 0; k < 3; ++k) {
    if (out.dims[k] < 2) throw Wfn1Error("load_system: inconsistent header: Grid: all dims must be >= 2");
    if (!(out.cell[k] > 0.0)) throw Wfn1Error("load_system: inconsistent header: Grid: cell lengths must be > 0");
  }
  const long long nr_declared = inum(at(doc, "nr"), "nr");
  out.n_v = static_cast<int>(inum(at(doc, "nv"), "nv"));
  out.n_c = static_cast<int>(inum(at(doc, "nc"), "nc"));
  out.n_r = static_cast<long long>(out.dims[0]) * out.dims[1] * out.dims[2];
  if (nr_declared != out.n_r) throw Wfn1Error("load_system: header nr does not match dims product");
  if (out.n_v < 1 || out.n_c < 1 || out.n_v + out.n_c > out.n_r)
    throw Wfn1Error("load_system: inconsistent header band counts");
  out.payload_offset = 8 + static_cast<long long>(len);
  return out;
}

void wfn1_read_payload(const char* path, long long offset, double* dst, size_t n, const char* what) {
  Fd f;
  f.fd = ::open(path, O_RDONLY);
  if (f.fd < 0) throw Wfn1Error(std::string("load_system: cannot open ") + path);
  char* p = reinterpret_cast<char*>(dst);
  size_t left = n * sizeof(double);
  off_t off = static_cast<off_t>(offset);
  while (left > 0) {
    const ssize_t r = ::pread(f.fd, p, left > (1u << 30) ? (1u << 30) : left, off);
    if (r <= 0) throw Wfn1Error(std::string("load_system: truncated payload reading ") + what);
    p += r;
    off += r;
    left -= static_cast<size_t>(r);
  }
}

void wfn1_write(const char* path, const int dims[3], const double cell[3], int n_v, int n_c, const double* psi,
                const double* energies, const double* vxc) {
  std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "wb"), &std::fclose);
  if (!f) throw Wfn1Error(std::string("save_system: cannot open ") + path);
  const std::string h = wfn1_header_json(dims, cell, n_v, n_c);
  const uint32_t len = static_cast<uint32_t>(h.size());
  const unsigned char lb[4] = {static_cast<unsigned char>(len & 0xff), static_cast<unsigned char>((len >> 8) & 0xff),
                               static_cast<unsigned char>((len >> 16) & 0xff),
                               static_cast<unsigned char>((len >> 24) & 0xff)};
  const size_t n_r = static_cast<size_t>(dims[0]) * dims[1] * dims[2];
  const size_t nb = static_cast<size_t>(n_v) + n_c;
  bool ok = std::fwrite("WFN1", 1, 4, f.get()) == 4 && std::fwrite(lb, 1, 4, f.get()) == 4 &&
            std::fwrite(h.data(), 1, h.size(), f.get()) == h.size();
  ok = ok && (n_r * nb == 0 || std::fwrite(psi, sizeof(double), n_r * nb, f.get()) == n_r * nb);
  ok = ok && (nb == 0 || std::fwrite(energies, sizeof(double), nb, f.get()) == nb);
  ok = ok && (nb == 0 || std::fwrite(vxc, sizeof(double), nb, f.get()) == nb);
  ok = ok && std::fflush(f.get()) == 0;
  if (!ok) throw Wfn1Error(std::string("save_system: write failed for ") + path);
}

}  // namespace lrgw_host
