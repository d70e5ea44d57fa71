// leo_front.cpp — native listing front-end (include/leo_front.h).
//
// One pass from listing text to the structure-of-arrays of include/leo_b200.h:
// the grammar and checks of disasm.parse_listing (disasm.py:259-409), the
// basic-block reconstruction of disasm.build_cfg (disasm.py:495-607) and the
// flattening of soa.encode_cfg.  Messages and their order follow the
// reference's ListingError / diagnostics text exactly (errors.py:15-30).
#include "../../include/leo_front.h"

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

enum Dialect { NVIDIA = 0, AMD = 1, INTEL = 2 };
// enums.py orders
enum RC { RC_VGPR = 0, RC_SGPR, RC_PRED, RC_BAR, RC_UNIFORM };
enum OC {
  GLOBAL_LOAD = 0, GLOBAL_STORE, LOCAL_LOAD, LOCAL_STORE, SCALAR_LOAD, CONSTANT_LOAD, ATOMIC, FP_ARITH,
  INT_ARITH, CONVERSION, CONTROL_FLOW, SYNC_WAIT, BARRIER_ALL, SEND, NOP, OTHER
};
const char* const kOcNames[] = {"global_load", "global_store", "local_load", "local_store", "scalar_load",
                                "constant_load", "atomic", "fp_arith", "int_arith", "conversion",
                                "control_flow", "sync_wait", "barrier_all", "send", "nop", "other"};
constexpr uint32_t kNone = 0xFFFFFFFFu;

bool is_load_class(int c) { return c == GLOBAL_LOAD || c == LOCAL_LOAD || c == SCALAR_LOAD || c == CONSTANT_LOAD; }
bool source_only(int c) {          // disasm.py _SOURCE_ONLY_CLASSES
  return c == GLOBAL_STORE || c == LOCAL_STORE || c == CONTROL_FLOW || c == SYNC_WAIT || c == BARRIER_ALL ||
         c == NOP;
}

// ---- Python string semantics (ASCII) -----------------------------------------
bool py_space(unsigned char c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f); }
bool word(unsigned char c) { return std::isalnum(c) || c == '_'; }
bool digit(unsigned char c) { return c >= '0' && c <= '9'; }
bool ident_start(unsigned char c) { return std::isalpha(c) || c == '_'; }

std::string strip(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && py_space(s[a])) a++;
  while (b > a && py_space(s[b - 1])) b--;
  return s.substr(a, b - a);
}
std::string rstrip(const std::string& s) {
  size_t b = s.size();
  while (b > 0 && py_space(s[b - 1])) b--;
  return s.substr(0, b);
}
std::string lower(std::string s) {
  for (auto& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}
std::vector<std::string> split_ws(const std::string& s) {   // str.split()
  std::vector<std::string> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && py_space(s[i])) i++;
    size_t j = i;
    while (j < s.size() && !py_space(s[j])) j++;
    if (j > i) out.push_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}
std::vector<std::string> splitlines(const std::string& t) {   // str.splitlines() (ASCII breaks)
  std::vector<std::string> out;
  out.reserve(t.size() / 32 + 16);
  size_t i = 0, n = t.size();
  while (i < n) {
    size_t j = i;
    while (j < n && !(t[j] == '\n' || t[j] == '\r' || t[j] == '\v' || t[j] == '\f' ||
                      (t[j] >= 0x1c && t[j] <= 0x1e)))
      j++;
    out.push_back(t.substr(i, j - i));
    if (j < n && t[j] == '\r' && j + 1 < n && t[j + 1] == '\n') j++;
    i = j + 1;
  }
  return out;
}
std::string py_repr(const std::string& s) {
  const bool sq = s.find('\'') != std::string::npos, dq = s.find('"') != std::string::npos;
  const char q = (sq && !dq) ? '"' : '\'';
  std::string o(1, q);
  for (unsigned char c : s) {
    if (c == '\\') o += "\\\\";
    else if (c == (unsigned char)q) { o += '\\'; o += (char)c; }
    else if (c == '\t') o += "\\t";
    else if (c == '\n') o += "\\n";
    else if (c == '\r') o += "\\r";
    else if (c < 0x20 || c == 0x7f) { char b[8]; snprintf(b, sizeof b, "\\x%02x", c); o += b; }
    else o += (char)c;
  }
  return o + q;
}
std::string hex(uint64_t v) { char b[32]; snprintf(b, sizeof b, "%llx", (unsigned long long)v); return b; }

struct ListingError : std::runtime_error {
  explicit ListingError(const std::string& m) : std::runtime_error(m) {}
};
[[noreturn]] void fail(const std::string& msg, long line = -1, long col = -1, const std::string& tok = "") {
  std::string where;
  if (line >= 0) {
    where = "line " + std::to_string(line);
    if (col >= 0) where += ", col " + std::to_string(col);
    where = " (" + where + ")";
  }
  const std::string t = tok.empty() ? "" : " near " + py_repr(tok);
  throw ListingError(msg + t + where);
}

// digits -> int64 (saturating past the SoA range; such values are rejected later)
int64_t to_int(const std::string& s, int base = 10) {
  int64_t v = 0;
  for (char c : s) {
    const int d = digit(c) ? c - '0' : (std::tolower(c) - 'a' + 10);
    if (v > (INT64_MAX - d) / base) return INT64_MAX;
    v = v * base + d;
  }
  return v;
}

// ---- opcode table (isa.py OpcodeTable) ------------------------------------------
struct OpTable {
  std::unordered_map<std::string, int> e;
  size_t max_len = 0;
  void parse(const std::string& text) {
    std::vector<std::pair<std::string, int>> entries;
    long ln = 0;
    for (const auto& raw : splitlines(text)) {
      ln++;
      const std::string line = strip(raw.substr(0, raw.find('#')));
      if (line.empty()) continue;
      const auto parts = split_ws(line);
      if (parts.size() != 2)
        throw ListingError("opcode table line " + std::to_string(ln) + ": expected '<pattern> <class>', got " +
                           py_repr(raw));
      int cls = -1;
      for (int c = 0; c < 16; c++) if (parts[1] == kOcNames[c]) cls = c;
      if (cls < 0)
        throw ListingError("opcode table line " + std::to_string(ln) + ": unknown opcode class " +
                           py_repr(parts[1]));
      entries.emplace_back(parts[0], cls);
    }
    // Python dict semantics: `entries[pattern] = cls` keeps the first
    // insertion position and the last value; the lowercase re-keying then
    // iterates in that order (isa.py OpcodeTable.__init__)
    std::vector<std::string> order;
    std::unordered_map<std::string, int> dict;
    for (auto& kv : entries) {
      if (!dict.count(kv.first)) order.push_back(kv.first);
      dict[kv.first] = kv.second;
    }
    for (const auto& key : order) e[lower(key)] = dict[key];
    for (auto& kv : e) max_len = std::max(max_len, kv.first.size());
  }
  int classify(const std::string& mn) const {
    thread_local std::string m, key;
    m = mn;
    for (auto& c : m) c = (char)std::tolower((unsigned char)c);
    for (size_t len = std::min(m.size(), max_len); len > 0; len--) {
      key.assign(m, 0, len);                      // reuses the buffer
      auto it = e.find(key);
      if (it != e.end()) return it->second;
    }
    return OTHER;
  }
};

// ---- decoded instruction ----------------------------------------------------------
struct Reg { int rc; int64_t index; int64_t span; };
struct Instr {
  int64_t offset;
  std::string mnemonic;
  int oc;
  std::vector<Reg> dests, srcs;
  bool has_guard = false;
  Reg guard{};
  int sync_kind = 0;
  uint32_t sync_a = kNone, sync_b = kNone;
  bool has_loc = false;
  std::string loc_str, loc_key;
  bool has_target = false;
  std::string target;
  std::vector<std::string> labels;
  std::string base_lower() const { return lower(mnemonic.substr(0, mnemonic.find('.'))); }
};

struct Kernel {
  std::string name;
  std::vector<Instr> ins;
  // cfg + SoA
  std::vector<uint8_t> opclass, sync_kind;
  std::vector<int32_t> block_of, opnd_ptr, blk_first, blk_last, succ_ptr, succ, pred_ptr, pred, line_id;
  std::vector<uint32_t> opnd, sync_a, sync_b;
  std::vector<int64_t> offset;
  int32_t unit_base[8] = {0};
  int64_t n_units = 0;
  std::vector<std::string> lines, diags;
};

// operand token kinds
struct Opnd { int kind; Reg reg; bool explicit_span; std::string text; int cnt; int64_t val; };
enum { K_REG, K_IMM, K_IDENT, K_CNT };

bool match_digits(const std::string& s, size_t& i) {
  const size_t a = i;
  while (i < s.size() && digit(s[i])) i++;
  return i > a;
}

Opnd parse_operand(int d, const std::string& t, long ln, long col) {
  Opnd o{};

  auto reg_plus = [&](int rc, size_t start, bool allow_plus) -> bool {
    // <prefix>(\d+)(:\+(\d+))?$
    size_t j = start;
    if (!match_digits(t, j)) return false;
    const std::string idx = t.substr(start, j - start);
    int64_t extra = 0;
    bool ex = false;
    if (j < t.size()) {
      if (!allow_plus || j + 2 > t.size() || t[j] != ':' || t[j + 1] != '+') return false;
      size_t k = j + 2;
      if (!match_digits(t, k) || k != t.size()) return false;
      extra = to_int(t.substr(j + 2, k - j - 2));
      ex = true;
    }
    o.kind = K_REG; o.reg = Reg{rc, to_int(idx), 1 + extra}; o.explicit_span = ex;
    return true;
  };
  auto single = [&](char p, size_t& j) -> bool {    // ^P(\d+)$ etc.
    if (t.empty() || t[0] != p) return false;
    j = 1;
    return match_digits(t, j) && j == t.size();
  };
  size_t j = 0;
  if (d == NVIDIA) {
    if (t.size() >= 2 && t[0] == 'U' && t[1] == 'R' && reg_plus(RC_UNIFORM, 2, true)) return o;
    if (!t.empty() && t[0] == 'R' && reg_plus(RC_VGPR, 1, true)) return o;
    if (single('P', j)) {
      const int64_t idx = to_int(t.substr(1));
      if (idx > 6) fail("predicate index out of range [0,6]", ln, col, t);
      o.kind = K_REG; o.reg = Reg{RC_PRED, idx, 1}; o.explicit_span = true;
      return o;
    }
    if (single('B', j)) {
      const int64_t idx = to_int(t.substr(1));
      if (idx < 1 || idx > 6) fail("barrier index out of range [1,6]", ln, col, t);
      o.kind = K_REG; o.reg = Reg{RC_BAR, idx, 1}; o.explicit_span = true;
      return o;
    }
  } else if (d == AMD) {
    for (const char* cn : {"vmcnt", "lgkmcnt"}) {
      const size_t L = strlen(cn);
      if (t.compare(0, L, cn) == 0 && t.size() > L + 2 && t[L] == '(' && t.back() == ')') {
        size_t k = L + 1;
        if (match_digits(t, k) && k == t.size() - 1) {
          o.kind = K_CNT; o.cnt = cn[0] == 'v' ? 0 : 1; o.val = to_int(t.substr(L + 1, k - L - 1));
          return o;
        }
      }
    }
    if (!t.empty() && (t[0] == 'v' || t[0] == 's')) {
      const int rc = t[0] == 'v' ? RC_VGPR : RC_SGPR;
      if (t.size() > 1 && t[1] == '[') {
        size_t k = 2;
        if (match_digits(t, k) && k < t.size() && t[k] == ':') {
          const size_t a = k + 1;
          size_t k2 = a;
          if (match_digits(t, k2) && k2 == t.size() - 1 && t.back() == ']') {
            const int64_t lo = to_int(t.substr(2, k - 2)), hi = to_int(t.substr(a, k2 - a));
            if (hi < lo) fail("register range is reversed", ln, col, t);
            o.kind = K_REG; o.reg = Reg{rc, lo, hi - lo + 1}; o.explicit_span = true;
            return o;
          }
        }
      } else {
        size_t k = 1;
        if (match_digits(t, k) && k == t.size()) {
          o.kind = K_REG; o.reg = Reg{rc, to_int(t.substr(1)), 1}; o.explicit_span = true;
          return o;
        }
      }
    }
    if (single('P', j)) { o.kind = K_REG; o.reg = Reg{RC_PRED, to_int(t.substr(1)), 1}; o.explicit_span = true; return o; }
  } else {
    if (!t.empty() && t[0] == 'r' && reg_plus(RC_VGPR, 1, true)) return o;
    if (single('P', j)) { o.kind = K_REG; o.reg = Reg{RC_PRED, to_int(t.substr(1)), 1}; o.explicit_span = true; return o; }
  }
  // immediates ^-?(?:0[xX][0-9a-fA-F]+|\d+)$
  {
    size_t k = (!t.empty() && t[0] == '-') ? 1 : 0;
    bool ok = false;
    if (t.size() > k + 2 && t[k] == '0' && (t[k + 1] == 'x' || t[k + 1] == 'X')) {
      size_t m = k + 2;
      while (m < t.size() && std::isxdigit((unsigned char)t[m])) m++;
      ok = m == t.size();
    }
    if (!ok) { size_t m = k; ok = match_digits(t, m) && m == t.size(); }
    if (ok) { o.kind = K_IMM; return o; }
  }
  // identifiers ^[A-Za-z_][\w.$]*$
  if (!t.empty() && ident_start(t[0])) {
    bool ok = true;
    for (size_t k = 1; k < t.size(); k++) if (!(word(t[k]) || t[k] == '.' || t[k] == '$')) ok = false;
    if (ok) { o.kind = K_IDENT; o.text = t; return o; }
  }
  fail("unrecognized operand", ln, col, t);
}

uint32_t parse_barrier_list(const std::string& v, long ln, long col) {
  uint32_t m = 0;
  size_t a = 0;
  while (true) {
    const size_t c = v.find(',', a);
    const std::string item = v.substr(a, c == std::string::npos ? std::string::npos : c - a);
    size_t k = 1;
    if (item.empty() || item[0] != 'B' || !match_digits(item, k) || k != item.size())
      fail("expected barrier list like B1,B3", ln, col, item);
    const int64_t idx = to_int(item.substr(1));
    if (idx < 1 || idx > 6) fail("barrier index out of range [1,6]", ln, col, item);
    m |= 1u << idx;
    if (c == std::string::npos) break;
    a = c + 1;
  }
  return m;
}
uint32_t parse_sbid_list(const std::string& v, long ln, long col) {
  uint32_t m = 0;
  size_t a = 0;
  while (true) {
    const size_t c = v.find(',', a);
    const std::string item = v.substr(a, c == std::string::npos ? std::string::npos : c - a);
    size_t k = 0;
    if (!match_digits(item, k) || k != item.size()) fail("expected sbid token list like 3,7", ln, col, item);
    const int64_t idx = to_int(item);
    if (idx > 31) fail("sbid token out of range [0,31]", ln, col, item);
    m |= 1u << idx;
    if (c == std::string::npos) break;
    a = c + 1;
  }
  return m;
}

// `{...}` annotation block (disasm.py:161-213) -> sync fields
void parse_annotations(int d, const std::string& body, long ln, long col, Instr& in) {
  uint32_t wait = 0, read = 0, write = 0, dep = 0, dst = 0, src = 0;
  int64_t stall = -1, set = -1;
  bool nv = false, intel = false;
  for (const auto& item : split_ws(body)) {
    const size_t eq = item.find('=');
    if (eq == std::string::npos) fail("annotation must be key=value", ln, col, item);
    const std::string key = item.substr(0, eq), val = item.substr(eq + 1);
    auto all_digits = [](const std::string& s) {
      if (s.empty()) return false;
      for (char c : s) if (!digit(c)) return false;
      return true;
    };
    if (key == "wait" || key == "read" || key == "write" || key == "depbar") {
      if (d != NVIDIA) fail(key + "= annotation is nvidia-only", ln, col, item);
      const uint32_t m = parse_barrier_list(val, ln, col);
      (key == "wait" ? wait : key == "read" ? read : key == "write" ? write : dep) |= m;
      nv = true;
    } else if (key == "stall") {
      if (d != NVIDIA) fail("stall= annotation is nvidia-only", ln, col, item);
      if (!all_digits(val)) fail("stall= expects a nonnegative integer", ln, col, item);
      stall = to_int(val);
      nv = true;
    } else if (key == "sbid.set") {
      if (d != INTEL) fail("sbid annotations are intel-only", ln, col, item);
      if (!all_digits(val) || to_int(val) > 31) fail("sbid token out of range [0,31]", ln, col, item);
      set = to_int(val);
      intel = true;
    } else if (key == "sbid.wait.dst" || key == "sbid.wait.src") {
      if (d != INTEL) fail("sbid annotations are intel-only", ln, col, item);
      (key == "sbid.wait.dst" ? dst : src) |= parse_sbid_list(val, ln, col);
      intel = true;
    } else {
      fail("unknown sync annotation", ln, col, item);
    }
  }
  if (nv) {
    if (stall >= (int64_t)kNone) fail("stall= value out of range", ln, col);
    in.sync_kind = 2;
    in.sync_a = write | (read << 8) | ((wait | dep) << 16);
    in.sync_b = stall < 0 ? kNone : (uint32_t)stall;
  } else if (intel) {
    in.sync_kind = 3;
    in.sync_a = set < 0 ? kNone : (uint32_t)set;
    in.sync_b = dst | src;
  }
}

// `file:line <- file:line ...` (disasm.py:216-228): all parts must parse
bool parse_src_loc(const std::string& comment, std::string& str, std::string& key) {
  std::vector<std::pair<std::string, std::string>> locs;
  size_t a = 0;
  while (true) {
    const size_t c = comment.find("<-", a);
    const std::string part = strip(comment.substr(a, c == std::string::npos ? std::string::npos : c - a));
    const size_t colon = part.rfind(':');
    if (colon == std::string::npos || colon == 0) return false;
    const std::string file = part.substr(0, colon), line = part.substr(colon + 1);
    for (char ch : file) if (py_space(ch) || ch == ':') return false;
    size_t k = 0;
    if (!match_digits(line, k) || k != line.size()) return false;
    locs.emplace_back(file, std::to_string(to_int(line)));
    if (c == std::string::npos) break;
    a = c + 2;
  }
  if (locs.empty()) return false;
  key = locs[0].first + ":" + locs[0].second;
  str = key;
  for (size_t i = 1; i < locs.size(); i++) str += " <- " + locs[i].first + ":" + locs[i].second;
  return true;
}

bool kernel_line(const std::string& line, std::string& name) {   // ^\.kernel\s+(name)\s*$
  if (line.compare(0, 7, ".kernel") != 0) return false;
  size_t i = 7;
  const size_t ws = i;
  while (i < line.size() && py_space(line[i])) i++;
  if (i == ws || i >= line.size() || !ident_start(line[i])) return false;
  const size_t a = i++;
  while (i < line.size() && (word(line[i]) || line[i] == '.' || line[i] == '$')) i++;
  name = line.substr(a, i - a);
  while (i < line.size() && py_space(line[i])) i++;
  return i == line.size();
}
bool label_line(const std::string& line, std::string& label) {     // ^(ident):\s*$
  if (line.empty() || !ident_start(line[0])) return false;
  size_t i = 1;
  while (i < line.size() && (word(line[i]) || line[i] == '.' || line[i] == '$')) i++;
  if (i >= line.size() || line[i] != ':') return false;
  label = line.substr(0, i);
  i++;
  while (i < line.size() && py_space(line[i])) i++;
  return i == line.size();
}

std::vector<std::pair<std::string, std::vector<Instr>>> parse_listing(int d, const std::string& text,
                                                                        const OpTable& table) {
  std::vector<std::pair<std::string, std::vector<Instr>>> kernels;
  bool have = false;
  std::string cur_name;
  std::vector<Instr> cur;
  std::vector<std::string> pending;
  std::vector<int64_t> seen;     // strictly increasing (enforced below)
  int64_t last = -1;
  auto flush = [&]() {
    if (have) {
      if (!pending.empty()) fail("label " + py_repr(pending[0]) + " at end of kernel binds no instruction");
      kernels.emplace_back(cur_name, std::move(cur));
    }
    cur.clear(); pending.clear(); seen.clear(); last = -1;
  };
  long ln = 0;
  for (const auto& raw : splitlines(text)) {
    ln++;
    const std::string line = strip(raw);
    if (line.empty() || line[0] == '#' || line.compare(0, 2, "//") == 0) continue;
    std::string nm;
    if (kernel_line(line, nm)) { flush(); have = true; cur_name = nm; continue; }
    if (label_line(line, nm)) {
      if (!have) fail("label outside a .kernel section", ln, 1, nm);
      pending.push_back(nm);
      continue;
    }
    if (!have) fail("instruction outside a .kernel section", ln, 1, split_ws(line)[0]);
    std::string rest = line;
    long col = (long)raw.find(line) + 1;
    Instr in;
    std::string comment;
    bool has_comment = false;
    const size_t cpos = rest.find("//");
    if (cpos != std::string::npos) {
      comment = strip(rest.substr(cpos + 2));
      has_comment = true;
      rest = rstrip(rest.substr(0, cpos));
    }
    bool has_off = false;
    int64_t off = 0;
    if (rest.compare(0, 2, "/*") == 0) {                          // ^/\*([0-9a-fA-F]+)\*/\s*
      size_t k = 2;
      while (k < rest.size() && std::isxdigit((unsigned char)rest[k])) k++;
      if (k > 2 && rest.compare(k, 2, "*/") == 0) {
        const std::string h = rest.substr(2, k - 2);
        if (h.size() > 15) fail("offset out of range", ln, col);
        off = to_int(h, 16);
        k += 2;
        while (k < rest.size() && py_space(rest[k])) k++;
        has_off = true;
        col += (long)k;
        rest = rest.substr(k);
      }
    }
    if (!rest.empty() && rest[0] == '@') {                        // ^@(!?)P(\d+)\s+
      size_t k = 1;
      const bool neg = k < rest.size() && rest[k] == '!';
      if (neg) k++;
      if (k < rest.size() && rest[k] == 'P') {
        const size_t a = ++k;
        if (match_digits(rest, k) && k < rest.size() && py_space(rest[k])) {
          const int64_t idx = to_int(rest.substr(a, k - a));
          while (k < rest.size() && py_space(rest[k])) k++;
          if (d == NVIDIA && idx > 6) fail("guard predicate out of range [0,6]", ln, col, strip(rest.substr(0, k)));
          in.has_guard = true;
          in.guard = Reg{RC_PRED, idx, 1};
          col += (long)k;
          rest = rest.substr(k);
        }
      }
    }
    // mnemonic ^[A-Za-z_][\w.]*
    if (rest.empty() || !ident_start(rest[0])) {
      const auto sp = split_ws(rest);
      fail("expected a mnemonic", ln, col, sp.empty() ? "" : sp[0]);
    }
    size_t k = 1;
    while (k < rest.size() && (word(rest[k]) || rest[k] == '.')) k++;
    in.mnemonic = rest.substr(0, k);
    col += (long)k;
    rest = rest.substr(k);
    const size_t bpos = rest.find('{');
    bool annotated = false;
    if (bpos != std::string::npos) {
      const size_t epos = rest.find('}', bpos);
      if (epos == std::string::npos) fail("unterminated { annotation block", ln, col + (long)bpos, "{");
      parse_annotations(d, rest.substr(bpos + 1, epos - bpos - 1), ln, col + (long)bpos, in);
      annotated = in.sync_kind != 0;
      const std::string trailing = strip(rest.substr(epos + 1));
      if (!trailing.empty()) fail("unexpected text after } annotation block", ln, col + (long)epos, trailing);
      rest = rest.substr(0, bpos);
    }
    in.oc = table.classify(in.mnemonic);
    thread_local std::vector<std::pair<Reg, bool>> regs;
    regs.clear();
    int64_t vm = -1, lg = -1;
    {
      const std::string body = strip(rest);
      size_t i = 0;
      while (i <= body.size()) {                                  // re.split(r"[,\s]+")
        size_t j = i;
        while (j < body.size() && body[j] != ',' && !py_space(body[j])) j++;
        const std::string tok = body.substr(i, j - i);
        if (!tok.empty()) {
          const Opnd o = parse_operand(d, tok, ln, col);
          if (o.kind == K_REG) regs.emplace_back(o.reg, o.explicit_span);
          else if (o.kind == K_CNT) (o.cnt == 0 ? vm : lg) = o.val;
          else if (o.kind == K_IDENT && in.oc == CONTROL_FLOW) {
            if (in.has_target) fail("multiple branch targets", ln, col, tok);
            in.has_target = true;
            in.target = o.text;
          }
        }
        if (j >= body.size()) break;
        while (j < body.size() && (body[j] == ',' || py_space(body[j]))) j++;
        i = j;
      }
    }
    if (vm >= 0 || lg >= 0) {
      if (d != AMD) fail("waitcnt counters are amd-only", ln, col);
      if (annotated) fail("waitcnt cannot also carry { } annotations", ln, col);
      if (vm >= (int64_t)kNone || lg >= (int64_t)kNone) fail("waitcnt counter out of range", ln, col);
      in.sync_kind = 1;
      in.sync_a = vm < 0 ? kNone : (uint32_t)vm;
      in.sync_b = lg < 0 ? kNone : (uint32_t)lg;
    }
    // width inference (nvidia, disasm.py:231-253)
    if (d == NVIDIA) {
      std::vector<std::string> parts;
      {
        size_t a = 0;
        while (true) {
          const size_t c = in.mnemonic.find('.', a);
          parts.push_back(in.mnemonic.substr(a, c == std::string::npos ? std::string::npos : c - a));
          if (c == std::string::npos) break;
          a = c + 1;
        }
      }
      std::string p0 = parts[0];
      for (auto& c : p0) c = (char)std::toupper((unsigned char)c);
      const bool widen_all = in.oc == FP_ARITH && !p0.empty() && p0[0] == 'D';
      int64_t dest_span = 0;
      if (is_load_class(in.oc) || in.oc == ATOMIC) {
        const bool has64 = std::find(parts.begin() + 1, parts.end(), "64") != parts.end();
        const bool has128 = std::find(parts.begin() + 1, parts.end(), "128") != parts.end();
        dest_span = has64 ? 2 : has128 ? 4 : 0;
      }
      for (size_t p = 0; p < regs.size(); p++) {
        auto& r = regs[p];
        if (!r.second && r.first.rc == RC_VGPR) {
          if (widen_all) r.first.span = 2;
          else if (dest_span && p == 0) r.first.span = dest_span;
        }
      }
    }
    in.srcs.reserve(regs.size());
    if (source_only(in.oc) || regs.empty()) {
      for (auto& r : regs) in.srcs.push_back(r.first);
    } else {
      in.dests.push_back(regs[0].first);
      for (size_t p = 1; p < regs.size(); p++) in.srcs.push_back(regs[p].first);
    }
    if (!has_off) off = last + 1;
    if (off <= last) {
      if (std::binary_search(seen.begin(), seen.end(), off))
        fail("duplicate offset 0x" + hex((uint64_t)off), ln, col);
      fail("offset 0x" + hex((uint64_t)off) + " does not increase", ln, col);
    }
    seen.push_back(off);
    last = off;
    in.offset = off;
    if (in.oc == CONTROL_FLOW) {
      const std::string b = in.base_lower();
      if (b == "cal" || b == "call" || b == "calla" || b == "s_call") { in.has_target = false; in.target.clear(); }
    }
    if (has_comment) in.has_loc = parse_src_loc(comment, in.loc_str, in.loc_key);
    in.labels = std::move(pending);
    pending.clear();
    cur.push_back(std::move(in));
  }
  flush();
  if (kernels.empty()) fail("no .kernel section found");
  return kernels;
}

bool is_terminator(const Instr& i) {
  if (i.oc != CONTROL_FLOW) return false;
  const std::string b = i.base_lower();
  return b == "exit" || b == "ret" || b == "s_endpgm" || b == "eot";
}
bool is_call(const Instr& i) {
  if (i.oc != CONTROL_FLOW) return false;
  const std::string b = i.base_lower();
  return b == "cal" || b == "call" || b == "calla" || b == "s_call";
}
bool is_cond(const Instr& i) {
  return i.has_target && (i.has_guard || lower(i.mnemonic).find("cbranch") != std::string::npos);
}

// build_cfg (disasm.py:495-607) + encode_cfg
void build(Kernel& K) {
  auto& ins = K.ins;
  const int n = (int)ins.size();
  K.opnd.reserve((size_t)n * 4);
  if (n == 0) fail("kernel " + py_repr(K.name) + " has no instructions");
  std::unordered_map<std::string, int> labels;
  for (int i = 0; i < n; i++)
    for (const auto& l : ins[i].labels) {
      if (labels.count(l)) fail("duplicate label " + py_repr(l) + " in kernel " + py_repr(K.name));
      labels[l] = i;
    }
  std::set<int> leaders{0};
  for (int i = 0; i < n; i++) {
    if (ins[i].has_target) {
      auto it = labels.find(ins[i].target);
      if (it == labels.end())
        fail("branch to unknown label " + py_repr(ins[i].target) + " at offset 0x" + hex((uint64_t)ins[i].offset));
      leaders.insert(it->second);
    }
    if (ins[i].oc == CONTROL_FLOW && i + 1 < n) leaders.insert(i + 1);
  }
  std::vector<int> starts(leaders.begin(), leaders.end());
  const int B = (int)starts.size();
  K.block_of.assign(n, 0);
  K.blk_first.resize(B);
  K.blk_last.resize(B);
  for (int b = 0; b < B; b++) {
    K.blk_first[b] = starts[b];
    K.blk_last[b] = b + 1 < B ? starts[b + 1] - 1 : n - 1;
    for (int i = K.blk_first[b]; i <= K.blk_last[b]; i++) K.block_of[i] = b;
  }
  std::vector<std::vector<int>> succs(B), preds(B);
  for (int b = 0; b < B; b++) {
    const Instr& l = ins[K.blk_last[b]];
    const int fall = b + 1 < B ? b + 1 : -1;
    std::vector<int> out;
    if (l.oc == CONTROL_FLOW) {
      if (is_terminator(l)) {
        if (l.has_guard && fall >= 0) out = {fall};
      } else if (is_call(l)) {
        if (fall >= 0) out = {fall};
      } else if (l.has_target) {
        const int tgt = K.block_of[labels[l.target]];
        if (is_cond(l)) {
          if (fall < 0 || tgt == fall) out = {tgt}; else out = {tgt, fall};
          if (fall < 0) K.diags.push_back("conditional branch at 0x" + hex((uint64_t)l.offset) +
                                          " has no fall-through instruction");
        } else {
          out = {tgt};
        }
      } else if (fall >= 0) {
        out = {fall};
      }
    } else if (fall >= 0) {
      out = {fall};
    } else {
      K.diags.push_back("kernel " + py_repr(K.name) + " does not end with a terminator; block " +
                        std::to_string(b) + " treated as exiting");
    }
    succs[b] = out;
  }
  for (int b = 0; b < B; b++) for (int s : succs[b]) preds[s].push_back(b);
  for (auto& p : preds) std::sort(p.begin(), p.end());
  std::vector<char> seen(B, 0);
  std::vector<int> st{0};
  seen[0] = 1;
  while (!st.empty()) {
    const int b = st.back(); st.pop_back();
    for (int s : succs[b]) if (!seen[s]) { seen[s] = 1; st.push_back(s); }
  }
  for (int b = 0; b < B; b++)
    if (!seen[b]) K.diags.push_back("block " + std::to_string(b) + " is unreachable from entry (retained)");
  K.succ_ptr.assign(B + 1, 0);
  K.pred_ptr.assign(B + 1, 0);
  for (int b = 0; b < B; b++) {
    K.succ.insert(K.succ.end(), succs[b].begin(), succs[b].end());
    K.pred.insert(K.pred.end(), preds[b].begin(), preds[b].end());
    K.succ_ptr[b + 1] = (int32_t)K.succ.size();
    K.pred_ptr[b + 1] = (int32_t)K.pred.size();
  }
  // SoA (soa.encode_cfg): operands srcs, guard, dests; units per class
  int64_t ext[8] = {0};
  K.opnd_ptr.assign(n + 1, 0);
  K.opclass.resize(n); K.sync_kind.resize(n); K.sync_a.resize(n); K.sync_b.resize(n);
  K.offset.resize(n); K.line_id.resize(n);
  std::unordered_map<std::string, int> line_tab;
  auto push = [&](int role, const Reg& r) {
    if (r.index < 0 || r.index >= 65536 || r.span < 1 || r.span >= 256)
      throw ListingError("register index/span out of SoA range: " + std::to_string(r.index) + "/" +
                         std::to_string(r.span));
    K.opnd.push_back((uint32_t)r.index | ((uint32_t)r.span << 16) | ((uint32_t)r.rc << 24) | ((uint32_t)role << 27));
    ext[r.rc] = std::max(ext[r.rc], r.index + r.span);
  };
  for (int i = 0; i < n; i++) {
    const Instr& x = ins[i];
    K.opclass[i] = (uint8_t)x.oc;
    K.offset[i] = x.offset;
    for (const auto& r : x.srcs) push(0, r);
    if (x.has_guard) push(1, x.guard);
    for (const auto& r : x.dests) push(2, r);
    K.opnd_ptr[i + 1] = (int32_t)K.opnd.size();
    K.sync_kind[i] = (uint8_t)x.sync_kind;
    K.sync_a[i] = x.sync_a;
    K.sync_b[i] = x.sync_b;
    const std::string key = x.has_loc ? x.loc_key : "<unknown>";
    auto it = line_tab.find(key);
    int lid;
    if (it == line_tab.end()) { lid = (int)K.lines.size(); line_tab[key] = lid; K.lines.push_back(key); }
    else lid = it->second;
    K.line_id[i] = lid;
  }
  int64_t acc = 0;
  for (int c = 0; c < 8; c++) { K.unit_base[c] = (int32_t)acc; acc += ext[c]; }
  K.n_units = acc;
}

struct Result {
  std::string error;
  std::vector<Kernel> kernels;
};

}  // namespace

extern "C" {

void* leo_front_parse(int32_t dialect, const char* text, int64_t len, const char* table_text, int64_t table_len) {
  auto* r = new Result();
  try {
    if (dialect < 0 || dialect > 2) throw ListingError("unknown dialect");
    OpTable table;
    table.parse(std::string(table_text ? table_text : "", table_text ? (size_t)table_len : 0));
    auto ks = parse_listing(dialect, std::string(text, (size_t)len), table);
    std::set<std::string> names;
    for (auto& kv : ks) {
      if (names.count(kv.first)) fail("duplicate kernel section " + py_repr(kv.first));
      names.insert(kv.first);
      Kernel K;
      K.name = kv.first;
      K.ins = std::move(kv.second);
      build(K);
      r->kernels.push_back(std::move(K));
    }
  } catch (const std::exception& e) {
    r->error = e.what();
    r->kernels.clear();
  }
  return r;
}

int32_t leo_front_error(void* h, char* buf, int32_t cap) {
  auto* r = (Result*)h;
  if (r->error.empty()) return 0;
  if (buf && cap > 0) {
    const size_t m = std::min((size_t)cap - 1, r->error.size());
    memcpy(buf, r->error.data(), m);
    buf[m] = 0;
  }
  return (int32_t)r->error.size();
}

int32_t leo_front_n_kernels(void* h) { return (int32_t)((Result*)h)->kernels.size(); }

const char* leo_front_kernel_name(void* h, int32_t k) { return ((Result*)h)->kernels.at(k).name.c_str(); }

int32_t leo_front_sizes(void* h, int32_t k, int64_t* s) {
  const Kernel& K = ((Result*)h)->kernels.at(k);
  s[0] = (int64_t)K.ins.size(); s[1] = (int64_t)K.blk_first.size(); s[2] = (int64_t)K.opnd.size();
  s[3] = (int64_t)K.succ.size(); s[4] = (int64_t)K.pred.size(); s[5] = K.n_units;
  s[6] = (int64_t)K.lines.size(); s[7] = (int64_t)K.diags.size();
  return 0;
}

int32_t leo_front_arrays(void* h, int32_t k, uint8_t* opclass, int32_t* block_of, int32_t* opnd_ptr,
                         uint32_t* opnd, uint8_t* sync_kind, uint32_t* sync_a, uint32_t* sync_b,
                         int32_t* blk_first, int32_t* blk_last, int32_t* succ_ptr, int32_t* succ,
                         int32_t* pred_ptr, int32_t* pred, int32_t* unit_base, int64_t* offset,
                         int32_t* line_id) {
  const Kernel& K = ((Result*)h)->kernels.at(k);
  auto cp = [](auto* dst, const auto& v) { if (!v.empty()) memcpy(dst, v.data(), v.size() * sizeof(v[0])); };
  cp(opclass, K.opclass); cp(block_of, K.block_of); cp(opnd_ptr, K.opnd_ptr); cp(opnd, K.opnd);
  cp(sync_kind, K.sync_kind); cp(sync_a, K.sync_a); cp(sync_b, K.sync_b); cp(blk_first, K.blk_first);
  cp(blk_last, K.blk_last); cp(succ_ptr, K.succ_ptr); cp(succ, K.succ); cp(pred_ptr, K.pred_ptr);
  cp(pred, K.pred); cp(offset, K.offset); cp(line_id, K.line_id);
  memcpy(unit_base, K.unit_base, sizeof(K.unit_base));
  return 0;
}

const char* leo_front_string(void* h, int32_t k, int32_t which, int32_t i) {
  const Kernel& K = ((Result*)h)->kernels.at(k);
  switch (which) {
    case 0: return K.ins.at(i).mnemonic.c_str();
    case 1: return K.ins.at(i).has_loc ? K.ins.at(i).loc_str.c_str() : nullptr;
    case 2: return K.lines.at(i).c_str();
    case 3: return K.diags.at(i).c_str();
  }
  return nullptr;
}

int64_t leo_front_strings(void* h, int32_t k, int32_t which, char* buf, int64_t cap) {
  const Kernel& K = ((Result*)h)->kernels.at(k);
  std::string out;
  const size_t n = which == 0 || which == 1 ? K.ins.size() : which == 2 ? K.lines.size() : K.diags.size();
  for (size_t i = 0; i < n; i++) {
    if (i) out += '\n';
    if (which == 0) out += K.ins[i].mnemonic;
    else if (which == 1) { if (K.ins[i].has_loc) out += K.ins[i].loc_str; }
    else if (which == 2) out += K.lines[i];
    else out += K.diags[i];
  }
  if (buf && cap >= (int64_t)out.size()) memcpy(buf, out.data(), out.size());
  return (int64_t)out.size();
}

void leo_front_free(void* h) { delete (Result*)h; }

}  // extern "C"
