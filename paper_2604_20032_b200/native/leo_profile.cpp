// leo_profile.cpp — native profile loader: profile JSON document -> ProfileSoA.
//
// Replaces the reference's profile front-end for the hot path's inputs:
//   profile.load_profiles  (profile.py:244-263)  JSON document -> KernelProfile list
//   profile._load_one      (profile.py:186-241)  schema checks, in the same order
//   InstructionSamples / KernelProfile __post_init__ (profile.py:124-165)
//   profile.attach         (profile.py:332-366)  offset join + skid diagnostics
//   soa.encode_profile     (dense per-instruction ProfileSoA arrays)
// in one C++ pass, without building per-record Python objects.
//
// The document is decoded exactly as CPython's json.JSONDecoder.raw_decode
// (the _json C scanner) decodes it, so malformed documents raise the same
// "malformed profile document: <msg>: line L column C (char P)" text, with
// positions counted in code points.  Values that appear in messages are
// formatted as Python's repr() formats them (str quoting, float shortest
// round-trip).  Deliberate differences, all on inputs the analysis path
// cannot use: integers outside int64 and counts that do not fit the SoA's
// int32 columns raise "value out of range"; non-integer stall counts raise
// "stall count must be an integer" (the reference compares or sums them and
// fails later, or with a TypeError); printable-ness in str repr follows the
// ASCII/Latin-1 rules only.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

using u32s = std::u32string;

// ---------------------------------------------------------------- UTF-8
// Strings are kept as UTF-8 bytes; code points are decoded only where a
// rule is per character (isspace, repr, positions in error messages).
int utf8_len(unsigned char c) {
  return c < 0x80 ? 1 : (c >> 5) == 6 ? 2 : (c >> 4) == 14 ? 3 : (c >> 3) == 30 ? 4 : 0;
}

bool utf8_valid(const char* p, int64_t n) {
  const auto* s = (const unsigned char*)p;
  for (int64_t i = 0; i < n;) {
    if (s[i] < 0x80) { i++; continue; }
    int len = utf8_len(s[i]);
    if (!len || i + len > n) return false;
    for (int k = 1; k < len; k++)
      if ((s[i + k] & 0xC0) != 0x80) return false;
    i += len;
  }
  return true;
}

uint32_t utf8_at(const unsigned char* s, int64_t i, int* len) {
  uint32_t c = s[i];
  *len = utf8_len(s[i]);
  if (*len > 1) {
    c &= (0x7F >> *len);
    for (int k = 1; k < *len; k++) c = (c << 6) | (s[i + k] & 0x3F);
  }
  return c;
}

u32s decode(const std::string& b) {
  u32s o;
  const auto* s = (const unsigned char*)b.data();
  for (int64_t i = 0; i < (int64_t)b.size();) {
    int len;
    o.push_back(utf8_at(s, i, &len));
    i += len ? len : 1;
  }
  return o;
}

void utf8_put(std::string& o, uint32_t c) {
  if (c < 0x80) o += (char)c;
  else if (c < 0x800) { o += (char)(0xC0 | (c >> 6)); o += (char)(0x80 | (c & 0x3F)); }
  else if (c < 0x10000) {
    o += (char)(0xE0 | (c >> 12)); o += (char)(0x80 | ((c >> 6) & 0x3F)); o += (char)(0x80 | (c & 0x3F));
  } else {
    o += (char)(0xF0 | (c >> 18)); o += (char)(0x80 | ((c >> 12) & 0x3F));
    o += (char)(0x80 | ((c >> 6) & 0x3F)); o += (char)(0x80 | (c & 0x3F));
  }
}

// str.isspace() (unicode White_Space with bidi WS/B/S or category Zs)
bool py_isspace(uint32_t c) {
  return (c >= 9 && c <= 13) || (c >= 0x1C && c <= 0x20) || c == 0x85 || c == 0xA0 ||
         c == 0x1680 || (c >= 0x2000 && c <= 0x200A) || c == 0x2028 || c == 0x2029 ||
         c == 0x202F || c == 0x205F || c == 0x3000;
}
bool json_ws(unsigned char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }

// ---------------------------------------------------------------- values
struct Scanner;

struct JVal {
  enum T { NUL, BOOL, INT, FLOAT, STR, ARR, OBJ } t = NUL;
  bool b = false;
  bool big = false;           // integer outside int64 (digits kept for repr)
  bool lazy = false;          // ARR / OBJ not materialised: bytes [a, z) of the document
  int64_t i = 0;
  double f = 0;
  int64_t a = 0, z = 0;
  std::string s;              // STR (UTF-8) or the big integer's digits
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;   // first-insertion order, last value wins
  std::vector<int64_t> starts;  // lazy ARR: byte offset of every element (recorded while validating)

  bool is_int() const { return t == INT || t == BOOL; }      // isinstance(x, int)
  int64_t ival() const { return t == BOOL ? (int64_t)b : i; }
  int sign() const { return t == BOOL ? (b ? 1 : 0) : big ? (s[0] == '-' ? -1 : 1) : (i > 0) - (i < 0); }
  const JVal* get(const char* k) const {
    const size_t n = strlen(k);
    for (auto& kv : obj)
      if (kv.first.size() == n && memcmp(kv.first.data(), k, n) == 0) return &kv.second;
    return nullptr;
  }
};

struct JsonError {
  std::string msg;
  int64_t pos;                // byte offset
};
struct StopIter {
  int64_t pos;
};

// CPython _json.c scanner semantics (scan_once_unicode, scanstring_unicode,
// _parse_object_unicode, _parse_array_unicode, _match_number_unicode), on
// UTF-8 bytes: every structural character is ASCII and a control character
// is a single byte, so the byte walk takes the same decisions as the code
// point walk; error positions are converted to code points when reported.
// Containers deeper than `depth` are validated but kept lazy (a byte span),
// so a million-record samples array is walked one record at a time.
struct Scanner {
  const unsigned char* s;
  int64_t n;
  Scanner(const char* t, int64_t len) : s((const unsigned char*)t), n(len) {}

  static int hexv(uint32_t c) {
    if (c >= '0' && c <= '9') return (int)(c - '0');
    if (c >= 'a' && c <= 'f') return (int)(c - 'a' + 10);
    if (c >= 'A' && c <= 'F') return (int)(c - 'A' + 10);
    return -1;
  }

  // `end` is the index after the opening quote; out == nullptr validates only
  int64_t scanstring(int64_t end, std::string* out) {
    const int64_t begin = end - 1;
    if (out) out->clear();
    for (;;) {
      unsigned char c = 0;
      int64_t next = end;
      for (; next < n; next++) {
        c = s[next];
        if (c == '"' || c == '\\') break;
        if (c <= 0x1f) throw JsonError{"Invalid control character at", next};
      }
      if (!(c == '"' || c == '\\') || next >= n) throw JsonError{"Unterminated string starting at", begin};
      if (out) out->append((const char*)s + end, (size_t)(next - end));
      next++;
      if (c == '"') return next;
      if (next == n) throw JsonError{"Unterminated string starting at", begin};
      uint32_t u = s[next];
      if (u != 'u') {
        end = next + 1;
        switch (u) {
          case '"': case '\\': case '/': break;
          case 'b': u = '\b'; break;
          case 'f': u = '\f'; break;
          case 'n': u = '\n'; break;
          case 'r': u = '\r'; break;
          case 't': u = '\t'; break;
          default: u = 0;
        }
        if (u == 0) throw JsonError{"Invalid \\escape", end - 2};
      } else {
        u = 0;
        next++;
        end = next + 4;
        if (end >= n) throw JsonError{"Invalid \\uXXXX escape", next - 1};
        for (; next < end; next++) {
          int h = hexv(s[next]);
          if (h < 0) throw JsonError{"Invalid \\uXXXX escape", end - 5};
          u = (u << 4) | (uint32_t)h;
        }
        if (u >= 0xD800 && u <= 0xDBFF && end + 6 < n && s[next++] == '\\' && s[next++] == 'u') {
          uint32_t c2 = 0;
          end += 6;
          for (; next < end; next++) {
            int h = hexv(s[next]);
            if (h < 0) throw JsonError{"Invalid \\uXXXX escape", end - 5};
            c2 = (c2 << 4) | (uint32_t)h;
          }
          if (c2 >= 0xDC00 && c2 <= 0xDFFF) u = 0x10000 + (((u - 0xD800) << 10) | (c2 - 0xDC00));
          else end -= 6;
        }
      }
      if (out) utf8_put(*out, u);   // a lone surrogate stays a (CESU-style) 3-byte unit
    }
  }

  bool lit(int64_t idx, const char* w) const {
    for (int64_t k = 0; w[k]; k++)
      if (s[idx + k] != (unsigned char)w[k]) return false;
    return true;
  }

  int64_t scan_once(int64_t idx, JVal* v, int depth) {
    if (idx < 0 || idx >= n) throw StopIter{idx};
    const unsigned char c = s[idx];
    if (!v) {   // validate only
      switch (c) {
        case '"': return scanstring(idx + 1, nullptr);
        case '{': return parse_object(idx + 1, nullptr, 0);
        case '[': return parse_array(idx + 1, nullptr, 0);
        case 'n': if (idx + 3 < n && lit(idx, "null")) return idx + 4; break;
        case 't': if (idx + 3 < n && lit(idx, "true")) return idx + 4; break;
        case 'f': if (idx + 4 < n && lit(idx, "false")) return idx + 5; break;
        case 'N': if (idx + 2 < n && lit(idx, "NaN")) return idx + 3; break;
        case 'I': if (idx + 7 < n && lit(idx, "Infinity")) return idx + 8; break;
        case '-': if (idx + 8 < n && lit(idx, "-Infinity")) return idx + 9; break;
      }
      return match_number(idx, nullptr);        // grammar only, no conversion
    }
    switch (c) {
      case '"': v->t = JVal::STR; return scanstring(idx + 1, &v->s);
      case '{':
      case '[': {
        v->t = c == '{' ? JVal::OBJ : JVal::ARR;
        if (depth <= 0) {
          const int64_t e = c == '{' ? parse_object(idx + 1, nullptr, 0)
                                     : parse_array(idx + 1, nullptr, 0, &v->starts);
          v->lazy = true; v->a = idx; v->z = e;
          return e;
        }
        return c == '{' ? parse_object(idx + 1, v, depth - 1) : parse_array(idx + 1, v, depth - 1);
      }
      case 'n':
        if (idx + 3 < n && lit(idx, "null")) { v->t = JVal::NUL; return idx + 4; }
        break;
      case 't':
        if (idx + 3 < n && lit(idx, "true")) { v->t = JVal::BOOL; v->b = true; return idx + 4; }
        break;
      case 'f':
        if (idx + 4 < n && lit(idx, "false")) { v->t = JVal::BOOL; v->b = false; return idx + 5; }
        break;
      case 'N':
        if (idx + 2 < n && lit(idx, "NaN")) { v->t = JVal::FLOAT; v->f = NAN; return idx + 3; }
        break;
      case 'I':
        if (idx + 7 < n && lit(idx, "Infinity")) { v->t = JVal::FLOAT; v->f = INFINITY; return idx + 8; }
        break;
      case '-':
        if (idx + 8 < n && lit(idx, "-Infinity")) { v->t = JVal::FLOAT; v->f = -INFINITY; return idx + 9; }
        break;
    }
    return match_number(idx, v);
  }

  static bool dig(unsigned char c) { return c >= '0' && c <= '9'; }

  int64_t match_number(int64_t start, JVal* vp) {
    const int64_t end_idx = n - 1;
    int64_t idx = start;
    bool is_float = false;
    if (s[idx] == '-') {
      idx++;
      if (idx > end_idx) throw StopIter{start};
    }
    if (s[idx] >= '1' && s[idx] <= '9') {
      idx++;
      while (idx <= end_idx && dig(s[idx])) idx++;
    } else if (s[idx] == '0') {
      idx++;
    } else {
      throw StopIter{start};
    }
    if (idx < end_idx && s[idx] == '.' && dig(s[idx + 1])) {
      is_float = true;
      idx += 2;
      while (idx <= end_idx && dig(s[idx])) idx++;
    }
    if (idx < end_idx && (s[idx] == 'e' || s[idx] == 'E')) {
      const int64_t e_start = idx;
      idx++;
      if (idx < end_idx && (s[idx] == '-' || s[idx] == '+')) idx++;
      while (idx <= end_idx && dig(s[idx])) idx++;
      if (dig(s[idx - 1])) is_float = true;
      else idx = e_start;
    }
    if (!vp) return idx;
    JVal& v = *vp;
    char buf[64];
    const int64_t len = idx - start;
    std::string big;
    const char* txt = buf;
    if (len < (int64_t)sizeof buf) {
      memcpy(buf, s + start, (size_t)len);
      buf[len] = 0;
    } else {
      big.assign((const char*)s + start, (size_t)len);
      txt = big.c_str();
    }
    if (is_float) {
      v.t = JVal::FLOAT;
      v.f = strtod(txt, nullptr);
    } else {
      v.t = JVal::INT;
      errno = 0;
      long long x = strtoll(txt, nullptr, 10);
      if (errno == ERANGE) {
        v.big = true;
        v.s = txt;
      } else {
        v.i = x;
      }
    }
    return idx;
  }

  int64_t parse_object(int64_t idx, JVal* v, int depth) {
    const int64_t end_idx = n - 1;
    std::unordered_map<std::string, size_t> pos;   // used once an object has many keys
    while (idx <= end_idx && json_ws(s[idx])) idx++;
    if (idx > end_idx || s[idx] != '}') {
      std::string key;
      for (;;) {
        if (idx > end_idx || s[idx] != '"')
          throw JsonError{"Expecting property name enclosed in double quotes", idx};
        idx = scanstring(idx + 1, v ? &key : nullptr);
        while (idx <= end_idx && json_ws(s[idx])) idx++;
        if (idx > end_idx || s[idx] != ':') throw JsonError{"Expecting ':' delimiter", idx};
        idx++;
        while (idx <= end_idx && json_ws(s[idx])) idx++;
        if (!v) {
          idx = scan_once(idx, nullptr, 0);
        } else {
          JVal val;
          idx = scan_once(idx, &val, depth);
          size_t at = v->obj.size();
          if (v->obj.size() < 16) {
            for (size_t k = 0; k < v->obj.size(); k++)
              if (v->obj[k].first == key) { at = k; break; }
          } else {
            if (pos.empty())
              for (size_t k = 0; k < v->obj.size(); k++) pos.emplace(v->obj[k].first, k);
            auto it = pos.find(key);
            if (it != pos.end()) at = it->second;
            else pos.emplace(key, v->obj.size());
          }
          if (at == v->obj.size()) v->obj.emplace_back(key, std::move(val));
          else v->obj[at].second = std::move(val);
        }
        while (idx <= end_idx && json_ws(s[idx])) idx++;
        if (idx <= end_idx && s[idx] == '}') break;
        if (idx > end_idx || s[idx] != ',') throw JsonError{"Expecting ',' delimiter", idx};
        idx++;
        while (idx <= end_idx && json_ws(s[idx])) idx++;
      }
    }
    return idx + 1;
  }

  int64_t parse_array(int64_t idx, JVal* v, int depth, std::vector<int64_t>* starts = nullptr) {
    const int64_t end_idx = n - 1;
    while (idx <= end_idx && json_ws(s[idx])) idx++;
    if (idx > end_idx || s[idx] != ']') {
      for (;;) {
        if (starts) starts->push_back(idx);
        if (v) {
          v->arr.emplace_back();
          idx = scan_once(idx, &v->arr.back(), depth);
        } else {
          idx = scan_once(idx, nullptr, 0);
        }
        while (idx <= end_idx && json_ws(s[idx])) idx++;
        if (idx <= end_idx && s[idx] == ']') break;
        if (idx > end_idx || s[idx] != ',') throw JsonError{"Expecting ',' delimiter", idx};
        idx++;
        while (idx <= end_idx && json_ws(s[idx])) idx++;
      }
    }
    return idx + 1;
  }

  // the fully materialised value of a lazy container (already validated)
  JVal materialize(const JVal& v) {
    if (!v.lazy) return v;
    JVal o;
    scan_once(v.a, &o, 1 << 20);
    return o;
  }

  // visit the elements of a (lazy or materialised) array, each materialised
  // `depth` levels deep
  template <class F>
  void for_each(const JVal& arr, int depth, F&& f) {
    if (!arr.lazy) {
      for (const JVal& e : arr.arr) f(e.lazy ? materialize(e) : e);
      return;
    }
    int64_t idx = arr.a + 1;
    while (json_ws(s[idx])) idx++;
    if (s[idx] == ']') return;
    JVal e;
    for (;;) {
      e = JVal();
      idx = scan_once(idx, &e, depth);
      f(e);
      while (json_ws(s[idx])) idx++;
      if (s[idx] == ']') return;
      idx++;
      while (json_ws(s[idx])) idx++;
    }
  }
};

thread_local Scanner* g_scan = nullptr;   // the document being loaded (repr of lazy values)

// ---------------------------------------------------------------- repr
std::string float_repr(double x) {
  if (std::isnan(x)) return "nan";
  if (std::isinf(x)) return x > 0 ? "inf" : "-inf";
  if (x == 0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  int prec = 1;
  for (; prec <= 17; prec++) {
    snprintf(buf, sizeof buf, "%.*e", prec - 1, x);
    if (strtod(buf, nullptr) == x) break;
  }
  // buf = [-]d.ddde[+-]XX
  std::string t(buf);
  bool neg = t[0] == '-';
  if (neg) t = t.substr(1);
  size_t epos = t.find('e');
  int exp10 = atoi(t.c_str() + epos + 1);
  std::string digs;
  for (size_t k = 0; k < epos; k++)
    if (t[k] != '.') digs += t[k];
  while (digs.size() > 1 && digs.back() == '0') digs.pop_back();
  const int decpt = exp10 + 1;   // digits d1 d2 ... with the point after decpt of them
  std::string o = neg ? "-" : "";
  if (decpt > -4 && decpt <= 16) {
    if (decpt <= 0) {
      o += "0.";
      o.append((size_t)(-decpt), '0');
      o += digs;
    } else if ((size_t)decpt >= digs.size()) {
      o += digs;
      o.append((size_t)decpt - digs.size(), '0');
      o += ".0";
    } else {
      o += digs.substr(0, (size_t)decpt) + "." + digs.substr((size_t)decpt);
    }
  } else {
    o += digs.substr(0, 1);
    if (digs.size() > 1) o += "." + digs.substr(1);
    char eb[16];
    snprintf(eb, sizeof eb, "e%c%02d", exp10 < 0 ? '-' : '+', std::abs(exp10));
    o += eb;
  }
  return o;
}

bool printable(uint32_t c) {
  if (c < 0x20 || c == 0x7F) return false;
  if (c >= 0x80 && c <= 0xA0) return false;
  if (c == 0xAD) return false;
  if (c >= 0xD800 && c <= 0xDFFF) return false;
  if (c == 0x2028 || c == 0x2029 || (c >= 0x2000 && c <= 0x200F) || c == 0xFEFF) return false;
  return true;
}

std::string str_repr(const std::string& b8) {
  const u32s s = decode(b8);
  bool has_sq = false, has_dq = false;
  for (uint32_t c : s) {
    has_sq |= c == '\'';
    has_dq |= c == '"';
  }
  const char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string o(1, q);
  char b[16];
  for (uint32_t c : s) {
    if (c == (uint32_t)q || c == '\\') { o += '\\'; o += (char)c; }
    else if (c == '\t') o += "\\t";
    else if (c == '\n') o += "\\n";
    else if (c == '\r') o += "\\r";
    else if (printable(c)) utf8_put(o, c);
    else if (c < 0x100) { snprintf(b, sizeof b, "\\x%02x", c); o += b; }
    else if (c < 0x10000) { snprintf(b, sizeof b, "\\u%04x", c); o += b; }
    else { snprintf(b, sizeof b, "\\U%08x", c); o += b; }
  }
  o += q;
  return o;
}

std::string repr(const JVal& v) {
  if (v.lazy) return repr(g_scan->materialize(v));
  switch (v.t) {
    case JVal::NUL: return "None";
    case JVal::BOOL: return v.b ? "True" : "False";
    case JVal::INT: return v.big ? v.s : std::to_string(v.i);
    case JVal::FLOAT: return float_repr(v.f);
    case JVal::STR: return str_repr(v.s);
    case JVal::ARR: {
      std::string o = "[";
      for (size_t k = 0; k < v.arr.size(); k++) o += (k ? ", " : "") + repr(v.arr[k]);
      return o + "]";
    }
    case JVal::OBJ: {
      std::string o = "{";
      for (size_t k = 0; k < v.obj.size(); k++)
        o += (k ? ", " : "") + str_repr(v.obj[k].first) + ": " + repr(v.obj[k].second);
      return o + "}";
    }
  }
  return "";
}

std::string py_str(const JVal& v) { return v.t == JVal::STR ? v.s : repr(v); }

std::string hexfmt(int64_t x) {   // f"{x:x}"
  char b[32];
  if (x < 0) snprintf(b, sizeof b, "-%llx", (unsigned long long)(-(x + 1)) + 1ull);
  else snprintf(b, sizeof b, "%llx", (unsigned long long)x);
  return b;
}

// ---------------------------------------------------------------- stall maps
// profile.py:52-99; common class index = CommonStall definition order
// (profile.py:29-43): memory_dep 0, execution_dep 1, synchronization 2,
// instruction_fetch 3, pipeline_busy 4, not_selected 5, idle 6, other 7.
struct Cat { const char* name; int cls; };
const Cat kNvidia[] = {
    {"instruction fetch", 3}, {"execution dependency", 1}, {"memory dependency", 0},
    {"texture", 0}, {"synchronization", 2}, {"constant memory dependency", 0},
    {"pipe busy", 4}, {"memory throttle", 0}, {"not selected", 5}, {"sleeping", 6},
    {"other", 7}, {nullptr, 0}};
const Cat kAmd[] = {
    {"no instruction available", 3}, {"alu dependency", 1}, {"waiting for memory", 0},
    {"internal instruction", 7}, {"barrier wait", 2}, {"not selected", 5},
    {"pipeline stall", 4}, {"sleep", 6}, {"other", 7}, {nullptr, 0}};
const Cat kIntel[] = {
    {"control flow", 7}, {"control flow stalls", 7}, {"controlstall", 7},
    {"pipeline hazards", 1}, {"pipestall", 1}, {"memory send operations", 0},
    {"sendstall", 0}, {"scoreboard id dependencies", 2}, {"sbidstall", 2},
    {"synchronization", 2}, {"syncstall", 2}, {"instruction fetch", 3},
    {"instrfetchstall", 3}, {"distribution stalls", 4}, {"diststall", 4},
    {"other stalls", 7}, {"otherstall", 7}, {nullptr, 0}};
const Cat* const kMaps[3] = {kNvidia, kAmd, kIntel};
const char* const kDialects[3] = {"nvidia", "amd", "intel"};

// " ".join(category.lower().split())  (profile.py:46-47), ASCII case folding
std::string norm_category(const std::string& c8) {
  std::string o;
  bool pending = false;
  for (uint32_t x : decode(c8)) {
    if (py_isspace(x)) { pending = !o.empty(); continue; }
    if (pending) { o += ' '; pending = false; }
    if (x >= 'A' && x <= 'Z') x += 32;
    utf8_put(o, x);
  }
  return o;
}

int map_stall(int dialect, const std::string& cat) {
  bool plain = true;     // fast path: lowercase ASCII without runs of spaces
  for (size_t x = 0; x < cat.size() && plain; x++) {
    const unsigned char ch = (unsigned char)cat[x];
    plain = (ch >= 'a' && ch <= 'z') || (ch == ' ' && x > 0 && x + 1 < cat.size() && cat[x - 1] != ' ');
  }
  bool ascii = true;
  for (unsigned char ch : cat) ascii &= ch < 0x80;
  std::string k;
  if (plain) k = cat;
  else if (ascii) {   // same as norm_category for ASCII text
    bool pending = false;
    for (unsigned char ch : cat) {
      if (ch == ' ' || (ch >= 9 && ch <= 13) || (ch >= 0x1C && ch <= 0x1F)) { pending = !k.empty(); continue; }
      if (pending) { k += ' '; pending = false; }
      k += (char)(ch >= 'A' && ch <= 'Z' ? ch + 32 : ch);
    }
  } else {
    k = norm_category(cat);
  }
  for (const Cat* c = kMaps[dialect]; c->name; c++)
    if (k == c->name) return c->cls;
  return -1;
}

// ---------------------------------------------------------------- records
struct Rec {
  int64_t offset, lat, total, exec;   // total / exec: -1 = None
  double eff;
  int64_t cls[8];
};
struct KProf {
  std::string name;
  int dialect = 0;
  int64_t period = 0;
  std::vector<Rec> recs;
};

// error kinds returned to the caller: 1 ProfileError, 2 InputError
// (unknown vendor, isa.Dialect.from_name), 3 value outside the SoA's range
struct ProfErr {
  int kind;
  std::string msg;
};

bool eq_ascii(const std::string& a, const char* k) { return a == k; }

// int(value, 16) for a str (Python int() grammar: surrounding whitespace,
// sign, optional 0x prefix, single underscores between digits)
bool parse_hex(const std::string& v8, int64_t* out) {
  const u32s v = decode(v8);
  size_t a = 0, b = v.size();
  while (a < b && py_isspace(v[a])) a++;
  while (b > a && py_isspace(v[b - 1])) b--;
  bool neg = false;
  if (a < b && (v[a] == '+' || v[a] == '-')) { neg = v[a] == '-'; a++; }
  bool prefixed = false;
  if (b - a >= 2 && v[a] == '0' && (v[a + 1] == 'x' || v[a + 1] == 'X')) { a += 2; prefixed = true; }
  if (a >= b) return false;
  unsigned __int128 x = 0;
  bool last_us = !prefixed;   // a leading '_' is allowed only right after the prefix
  bool any = false;
  for (size_t k = a; k < b; k++) {
    if (v[k] == '_') {
      if (last_us) return false;
      last_us = true;
      continue;
    }
    int h = Scanner::hexv(v[k]);
    if (h < 0) return false;
    x = x * 16 + (unsigned)h;
    if (x > ((unsigned __int128)1 << 64)) throw ProfErr{3, "offset value out of range"};
    last_us = false;
    any = true;
  }
  if (!any || last_us) return false;
  if (!neg && x > (unsigned __int128)INT64_MAX) throw ProfErr{3, "offset value out of range"};
  if (neg && x > (unsigned __int128)INT64_MAX + 1) throw ProfErr{3, "offset value out of range"};
  *out = neg ? (int64_t)(0 - (uint64_t)x) : (int64_t)x;
  return true;
}

std::string at_off(int64_t off) { return " at offset 0x" + hexfmt(off); }

int64_t need_i64(const JVal& v, const char* what) {
  if (v.big) throw ProfErr{3, std::string(what) + " value out of range"};
  return v.ival();
}

// profile._parse_offset (profile.py:172-183)
int64_t parse_offset(const JVal& v) {
  if (v.is_int()) {
    if (v.sign() < 0) throw ProfErr{1, "negative offset " + repr(v)};
    return need_i64(v, "offset");
  }
  if (v.t == JVal::STR) {
    int64_t o;
    if (!parse_hex(v.s, &o)) throw ProfErr{1, "offset " + repr(v) + " is not a hex string"};
    return o;
  }
  throw ProfErr{1, "offset must be a hex string, got " + repr(v)};
}

std::string sorted_join(std::vector<std::string> keys) {
  std::sort(keys.begin(), keys.end());
  std::string o;
  for (size_t k = 0; k < keys.size(); k++) o += (k ? ", " : "") + keys[k];
  return o;
}

// The records of a samples array, in document order.  A big lazy array is
// split at element boundaries over host threads; each record is checked in
// full by one thread, and the error reported is the first record's in
// document order (what the sequential loop would raise).
template <class F>
void load_records(const JVal& samples, F&& one, std::vector<Rec>& out) {
  Scanner* sc = g_scan;
  const std::vector<int64_t>& starts = samples.starts;   // element offsets, recorded by the validation
  const int64_t n = samples.lazy ? (int64_t)starts.size() : (int64_t)samples.arr.size();
  unsigned nt = std::thread::hardware_concurrency();
  nt = n < 16384 ? 1u : std::max(1u, std::min(nt, 32u));
  out.resize((size_t)n);
  std::vector<int64_t> err_at(nt, -1);
  std::vector<ProfErr> errs(nt);
  auto work = [&](unsigned w) {
    g_scan = sc;
    const int64_t lo = n * w / nt, hi = n * (w + 1) / nt;
    JVal e;
    for (int64_t t = lo; t < hi; t++) {
      try {
        if (samples.lazy) {
          e = JVal();
          sc->scan_once(starts[(size_t)t], &e, 1 << 20);
          out[(size_t)t] = one(e);
        } else {
          const JVal& x = samples.arr[(size_t)t];
          out[(size_t)t] = one(x.lazy ? sc->materialize(x) : x);
        }
      } catch (const ProfErr& pe) {
        err_at[w] = t;
        errs[w] = pe;
        return;
      }
    }
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nt; w++) th.emplace_back(work, w);
    for (auto& t : th) t.join();
  }
  for (unsigned w = 0; w < nt; w++)      // chunks are in order: the first failing chunk holds the first error
    if (err_at[w] >= 0) throw errs[w];
}

// profile._load_one (profile.py:186-241) with the __post_init__ checks of
// InstructionSamples (:124-144) and KernelProfile (:154-161) in order
KProf load_one(const JVal& obj) {
  if (obj.t != JVal::OBJ) throw ProfErr{1, "profile entry must be a JSON object"};
  static const char* req[] = {"kernel", "vendor", "period_cycles", "samples"};
  for (const char* k : req)
    if (!obj.get(k)) throw ProfErr{1, std::string("profile entry missing required field '") + k + "'"};
  {
    std::vector<std::string> unk;
    for (auto& kv : obj.obj) {
      bool known = false;
      for (const char* k : req) known |= eq_ascii(kv.first, k);
      if (!known) unk.push_back(kv.first);
    }
    if (!unk.empty()) throw ProfErr{1, "unknown profile field(s): " + sorted_join(unk)};
  }
  KProf kp;
  {   // Dialect.from_name(str(vendor)): name.strip().lower()  (isa.py:25-29)
    const JVal& vv = *obj.get("vendor");
    const std::string name = py_str(vv);
    const u32s raw = decode(name);
    size_t a = 0, b = raw.size();
    while (a < b && py_isspace(raw[a])) a++;
    while (b > a && py_isspace(raw[b - 1])) b--;
    std::string low;
    for (size_t k = a; k < b; k++) {
      uint32_t c = raw[k];
      if (c >= 'A' && c <= 'Z') c += 32;
      utf8_put(low, c);
    }
    int d = -1;
    for (int k = 0; k < 3; k++)
      if (low == kDialects[k]) d = k;
    if (d < 0) {
      throw ProfErr{2, "unknown vendor " + str_repr(name) + "; expected one of nvidia, amd, intel"};
    }
    kp.dialect = d;
  }
  const JVal& per = *obj.get("period_cycles");
  if (!per.is_int() || per.sign() <= 0)
    throw ProfErr{1, "period_cycles must be a positive integer, got " + repr(per)};
  kp.period = need_i64(per, "period_cycles");
  const JVal& samples = *obj.get("samples");
  if (samples.t != JVal::ARR) throw ProfErr{1, "samples must be an array"};
  static const char* rfields[] = {"offset", "counts", "latency_samples", "total_samples",
                                  "exec_count", "efficiency"};
  auto one = [&](const JVal& rec) -> Rec {
    if (rec.t != JVal::OBJ) throw ProfErr{1, "sample record must be a JSON object"};
    {
      std::vector<std::string> extra;
      for (auto& kv : rec.obj) {
        bool known = false;
        for (const char* k : rfields) known |= eq_ascii(kv.first, k);
        if (!known) extra.push_back(kv.first);
      }
      if (!extra.empty()) throw ProfErr{1, "unknown sample field(s): " + sorted_join(extra)};
    }
    for (int k = 0; k < 3; k++)
      if (!rec.get(rfields[k]))
        throw ProfErr{1, std::string("sample record missing required field '") + rfields[k] + "'"};
    Rec r{};
    r.offset = parse_offset(*rec.get("offset"));

    const JVal& counts = *rec.get("counts");
    if (counts.t != JVal::OBJ) throw ProfErr{1, "counts must be an object" + at_off(r.offset)};
    for (auto& kv : counts.obj)
      if (map_stall(kp.dialect, kv.first) < 0)
        throw ProfErr{1, std::string("unknown ") + kDialects[kp.dialect] + " stall category " +
                             str_repr(kv.first)};
    const JVal& lat = *rec.get("latency_samples");
    if (!lat.is_int()) throw ProfErr{1, "latency_samples must be an integer" + at_off(r.offset)};
    const JVal* tot = rec.get("total_samples");
    if (tot && tot->t == JVal::NUL) tot = nullptr;
    if (tot && !tot->is_int()) throw ProfErr{1, "total_samples must be an integer" + at_off(r.offset)};
    const JVal* ex = rec.get("exec_count");
    if (ex && ex->t == JVal::NUL) ex = nullptr;
    if (ex && !ex->is_int()) throw ProfErr{1, "exec_count must be an integer" + at_off(r.offset)};
    const JVal* ef = rec.get("efficiency");
    if (ef && !(ef->t == JVal::INT || ef->t == JVal::FLOAT))
      throw ProfErr{1, "efficiency must be a number" + at_off(r.offset)};
    // InstructionSamples.__post_init__
    if (lat.sign() < 0) throw ProfErr{1, "negative sample count" + at_off(r.offset)};
    if (tot) {
      if (tot->sign() < 0) throw ProfErr{1, "negative sample count" + at_off(r.offset)};
      r.total = need_i64(*tot, "total_samples");
    } else {
      r.total = -1;
    }
    r.lat = need_i64(lat, "latency_samples");
    if (tot && r.lat > r.total)
      throw ProfErr{1, "latency_samples " + repr(lat) + " > total_samples " + repr(*tot) + at_off(r.offset)};
    for (auto& kv : counts.obj) {
      const JVal& c = kv.second;
      if (!c.is_int()) throw ProfErr{3, "stall count must be an integer" + at_off(r.offset)};
      if (c.sign() < 0) throw ProfErr{1, "negative stall count" + at_off(r.offset)};
    }
    __int128 sum = 0;
    for (auto& kv : counts.obj) {
      const int64_t c = need_i64(kv.second, "stall count");
      sum += c;
      r.cls[map_stall(kp.dialect, kv.first)] += c;
    }
    if (sum != r.lat) {
      char b[48];
      snprintf(b, sizeof b, "%lld", (long long)sum);
      throw ProfErr{1, std::string("stall counts sum to ") + b + " but latency_samples is " +
                           repr(lat) + at_off(r.offset)};
    }
    if (ex) {
      if (ex->sign() < 0) throw ProfErr{1, "negative exec_count" + at_off(r.offset)};
      r.exec = need_i64(*ex, "exec_count");
    } else {
      r.exec = -1;
    }
    r.eff = 1.0;
    if (ef) r.eff = ef->t == JVal::FLOAT ? ef->f : ef->big ? strtod(ef->s.c_str(), nullptr) : (double)ef->i;
    if (!(0.0 < r.eff && r.eff <= 1.0))
      throw ProfErr{1, "efficiency must be in (0,1], got " + float_repr(r.eff)};
    return r;
  };
  load_records(samples, one, kp.recs);
  kp.name = py_str(*obj.get("kernel"));
  {   // KernelProfile.__post_init__: duplicate offsets, smallest reported
    std::vector<int64_t> offs;
    offs.reserve(kp.recs.size());
    for (auto& r : kp.recs) offs.push_back(r.offset);
    std::sort(offs.begin(), offs.end());
    for (size_t k = 1; k < offs.size(); k++)
      if (offs[k] == offs[k - 1]) throw ProfErr{1, "duplicate sample offset 0x" + hexfmt(offs[k])};
  }
  return kp;
}

struct Doc {
  int err_kind = 0;
  std::string err;
  std::vector<KProf> kernels;
  std::string diag;    // last attach's diagnostics
};

// JSONDecodeError's position text, in code points (json/decoder.py:35-40)
std::string pos_suffix(const char* text, int64_t pos) {
  int64_t line = 1, chars = 0, last_nl = -1;
  for (int64_t k = 0; k < pos; k++) {
    const unsigned char c = (unsigned char)text[k];
    if ((c & 0xC0) == 0x80) continue;
    if (c == '\n') { line++; last_nl = chars; }
    chars++;
  }
  const int64_t col = chars - last_nl;
  return ": line " + std::to_string(line) + " column " + std::to_string(col) + " (char " +
         std::to_string(chars) + ")";
}

// profile.load_profiles (profile.py:244-263)
void load_profiles(Doc& d, const char* text, int64_t n) {
  Scanner sc(text, n);
  g_scan = &sc;
  int64_t pos = 0;
  while (pos < n) {
    for (;;) {      // text[pos].isspace()
      if (pos >= n) break;
      int len;
      const uint32_t c = utf8_at(sc.s, pos, &len);
      if (!py_isspace(c)) break;
      pos += len;
    }
    if (pos >= n) break;
    JVal obj;
    try {
      pos = sc.scan_once(pos, &obj, 1);
    } catch (const JsonError& e) {
      throw ProfErr{1, "malformed profile document: " + e.msg + pos_suffix(text, e.pos)};
    } catch (const StopIter& e) {
      throw ProfErr{1, "malformed profile document: Expecting value" + pos_suffix(text, e.pos)};
    }
    d.kernels.push_back(load_one(obj));
  }
  if (d.kernels.empty()) throw ProfErr{1, "profile document contains no kernel objects"};
  std::vector<std::string> names;
  for (auto& k : d.kernels) names.push_back(k.name);
  std::sort(names.begin(), names.end());
  for (size_t k = 1; k < names.size(); k++)
    if (names[k] == names[k - 1]) throw ProfErr{1, "profile document has duplicate kernel entries"};
}

}  // namespace

extern "C" {

void* leo_profile_parse(const char* text, int64_t len) {
  auto* d = new Doc();
  if (!utf8_valid(text, len)) {
    d->err_kind = 1;
    d->err = "profile document is not valid UTF-8";
    return d;
  }
  try {
    load_profiles(*d, text, len);
  } catch (const ProfErr& e) {
    d->err_kind = e.kind;
    d->err = e.msg;
    d->kernels.clear();
  }
  return d;
}

/* error kind (0 none, 1 ProfileError, 2 InputError, 3 out of range); the
 * message is copied into buf (NUL-terminated) when cap > 0 */
int32_t leo_profile_error(void* h, char* buf, int32_t cap, int32_t* len) {
  auto* d = (Doc*)h;
  if (len) *len = (int32_t)d->err.size();
  if (buf && cap > 0) {
    size_t n = std::min((size_t)cap - 1, d->err.size());
    memcpy(buf, d->err.data(), n);
    buf[n] = 0;
  }
  return d->err_kind;
}

int32_t leo_profile_n_kernels(void* h) { return (int32_t)((Doc*)h)->kernels.size(); }

const char* leo_profile_kernel_name(void* h, int32_t k) { return ((Doc*)h)->kernels[k].name.c_str(); }

/* info[0..2] = dialect (0 nvidia, 1 amd, 2 intel), sampling period, record count */
int32_t leo_profile_info(void* h, int32_t k, int64_t* info) {
  auto& kp = ((Doc*)h)->kernels[k];
  info[0] = kp.dialect;
  info[1] = kp.period;
  info[2] = (int64_t)kp.recs.size();
  return 0;
}

/* kernel k's records in document order: offset, latency, total (-1 None),
 * exec (-1 None), efficiency, per-common-class counts [n, 8] */
int32_t leo_profile_records(void* h, int32_t k, int64_t* offset, int64_t* lat, int64_t* total,
                            int64_t* exec, double* eff, int64_t* cls) {
  auto& kp = ((Doc*)h)->kernels[k];
  for (size_t r = 0; r < kp.recs.size(); r++) {
    const Rec& x = kp.recs[r];
    offset[r] = x.offset; lat[r] = x.lat; total[r] = x.total; exec[r] = x.exec; eff[r] = x.eff;
    for (int c = 0; c < 8; c++) cls[r * 8 + c] = x.cls[c];
  }
  return 0;
}

/* profile.attach (profile.py:332-366) + soa.encode_profile: join kernel k's
 * records to the instructions by offset into the dense ProfileSoA columns
 * (lat i32[N], cls_cnt i32[N,8], exec i64[N] (-1 None), total i32[N] (-1
 * None), eff f64[N], sampled u8[N]).  Returns 0, or 1 (ProfileError) / 3 (a
 * value outside the i32 columns) with the message in leo_profile_error.  The
 * skid diagnostic (empty when none) is in leo_profile_diagnostic. */
int32_t leo_profile_attach(void* h, int32_t k, const char* cfg_name, int32_t cfg_dialect, int32_t n,
                           const int64_t* instr_offset, int32_t* lat, int32_t* cls, int64_t* exec,
                           int32_t* total, double* eff, uint8_t* sampled) {
  auto* d = (Doc*)h;
  auto& kp = d->kernels[k];
  d->diag.clear();
  d->err_kind = 0;
  d->err.clear();
  if (kp.name != cfg_name) {
    d->err_kind = 1;
    d->err = "profile kernel " + str_repr(kp.name) +
             " does not match disassembly kernel " + str_repr(std::string(cfg_name));
    return 1;
  }
  if (kp.dialect != cfg_dialect) {
    d->err_kind = 1;
    d->err = std::string("profile vendor ") + kDialects[kp.dialect] +
             " does not match disassembly dialect " + kDialects[cfg_dialect];
    return 1;
  }
  std::unordered_map<int64_t, int32_t> by_off;
  by_off.reserve((size_t)n * 2);
  for (int32_t i = 0; i < n; i++) by_off[instr_offset[i]] = i;   // last index wins, as the dict does
  for (int32_t i = 0; i < n; i++) {
    lat[i] = 0; total[i] = -1; exec[i] = -1; eff[i] = 1.0; sampled[i] = 0;
    for (int c = 0; c < 8; c++) cls[(size_t)i * 8 + c] = 0;
  }
  std::vector<int64_t> skid;
  for (const Rec& r : kp.recs) {
    auto it = by_off.find(r.offset);
    if (it == by_off.end()) { skid.push_back(r.offset); continue; }
    const int32_t i = it->second;
    if (r.lat > INT32_MAX || r.total > INT32_MAX) {
      d->err_kind = 3;
      d->err = "sample count out of range for the device layout" + at_off(r.offset);
      return 3;
    }
    lat[i] = (int32_t)r.lat;
    total[i] = (int32_t)r.total;
    exec[i] = r.exec;
    eff[i] = r.eff;
    sampled[i] = 1;
    for (int c = 0; c < 8; c++) cls[(size_t)i * 8 + c] = (int32_t)r.cls[c];
  }
  if (!skid.empty()) {
    std::sort(skid.begin(), skid.end());
    d->diag = std::to_string(skid.size()) + " sampled offset(s) match no instruction (skid): ";
    for (size_t x = 0; x < skid.size(); x++) d->diag += (x ? ", 0x" : "0x") + hexfmt(skid[x]);
  }
  return 0;
}

const char* leo_profile_diagnostic(void* h) { return ((Doc*)h)->diag.c_str(); }

void leo_profile_free(void* h) { delete (Doc*)h; }

}  // extern "C"
