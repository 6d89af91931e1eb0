// occx_sass.cpp -- native tokenizer for the reference's disassembly grammar
// (occmix/sass.py:216-339, README "Disassembly listing"), emitting the
// 4-byte K0 instruction records directly.
//
// Host C++; exactness goal: the same functions, instructions, errors and
// error line numbers as occmix.parse_disassembly on any str input.  The
// regexes are restated by hand on code points; \s \w \d and str.isspace /
// splitlines use tables generated from the running CPython
// (tools/gen_unicode_tables.py -> occx_unicode.h).  Reference quirks kept:
//   * a label-shaped line ("NAME:") starts a new function (sass.py:291-297);
//   * an opcode followed by a non-space separator (tab) or a second ';'
//     makes the reference raise AttributeError (sass.py:278-279 matches the
//     opcode regex on `body.partition(" ")[0]`): status OCCX_ERR_ATTRIBUTE.
// Record = OCCX_INSTR(signature id (interned opcode + modifiers), register
// operands (`\bR\d+\b` matches over the operand tokens,
// sass.py:57,84-88,105-107), predicate guard).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_map>
#include <functional>
#include <algorithm>
#include <thread>
#include <vector>

#include "../../include/occx.h"
#include "occx_unicode.h"

namespace {

bool in_ranges(const occx_uc::Range* r, uint32_t n, uint32_t c) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (c < r[mid].lo) hi = mid;
    else if (c > r[mid].hi) lo = mid + 1;
    else return true;
  }
  return false;
}

struct Classes {   // 0..255 cached, the rest by range search
  uint8_t space[256], word[256], digit[256];
  Classes() {
    for (uint32_t c = 0; c < 256; ++c) {
      space[c] = in_ranges(occx_uc::k_space, occx_uc::k_space_n, c);
      word[c] = in_ranges(occx_uc::k_word, occx_uc::k_word_n, c);
      digit[c] = in_ranges(occx_uc::k_digit, occx_uc::k_digit_n, c);
    }
  }
};
const Classes g_cls;                 // built at library load
inline bool is_space(uint32_t c) {   // re \s == str.isspace under CPython 3.12 (generator checks)
  return c < 256 ? g_cls.space[c] : in_ranges(occx_uc::k_space, occx_uc::k_space_n, c);
}
inline bool is_word(uint32_t c) {
  return c < 256 ? g_cls.word[c] : in_ranges(occx_uc::k_word, occx_uc::k_word_n, c);
}
inline bool is_digit(uint32_t c) {
  return c < 256 ? g_cls.digit[c] : in_ranges(occx_uc::k_digit, occx_uc::k_digit_n, c);
}
inline bool is_upper(uint32_t c) { return c >= 'A' && c <= 'Z'; }
inline bool is_upper_digit(uint32_t c) { return is_upper(c) || (c >= '0' && c <= '9'); }
inline bool is_hex(uint32_t c) {
  return (c >= '0' && c <= '9') || (c >= 'a' && c <= 'f') || (c >= 'A' && c <= 'F');
}

using Str = std::vector<uint32_t>;   // code points of one line

// view [b, e) into a line
struct View {
  const uint32_t* p;
  size_t b, e;
  size_t size() const { return e - b; }
  uint32_t operator[](size_t i) const { return p[b + i]; }
  bool empty() const { return b >= e; }
};

View strip(View v) {
  while (v.b < v.e && is_space(v.p[v.b])) ++v.b;
  while (v.e > v.b && is_space(v.p[v.e - 1])) --v.e;
  return v;
}
View rstrip(View v) {
  while (v.e > v.b && is_space(v.p[v.e - 1])) --v.e;
  return v;
}
bool starts_with(View v, const char* s) {
  size_t n = std::strlen(s);
  if (v.size() < n) return false;
  for (size_t i = 0; i < n; ++i)
    if (v[i] != (uint32_t)(unsigned char)s[i]) return false;
  return true;
}
size_t skip_ws(View v, size_t i) {
  while (i < v.size() && is_space(v[i])) ++i;
  return i;
}

// ^\s*([A-Za-z_$][\w$.@]*)\s*:\s*$  -> name range (relative) or false
bool label_match(View v, size_t* nb, size_t* ne) {
  size_t i = skip_ws(v, 0);
  if (i >= v.size()) return false;
  const uint32_t c0 = v[i];
  if (!((c0 >= 'A' && c0 <= 'Z') || (c0 >= 'a' && c0 <= 'z') || c0 == '_' || c0 == '$'))
    return false;
  size_t j = i + 1;
  while (j < v.size() && (is_word(v[j]) || v[j] == '$' || v[j] == '.' || v[j] == '@')) ++j;
  size_t k = skip_ws(v, j);
  if (k >= v.size() || v[k] != ':') return false;
  k = skip_ws(v, k + 1);
  if (k != v.size()) return false;
  if (nb) *nb = i;
  if (ne) *ne = j;
  return true;
}

// _function_header_name (sass.py:291-297)
bool header_name(View v, size_t* nb, size_t* ne) {
  // ^\s*Function\s*:\s*(\S+)\s*$
  {
    size_t i = skip_ws(v, 0);
    View w{v.p, v.b + i, v.e};
    if (starts_with(w, "Function")) {
      i = skip_ws(v, i + 8);
      if (i < v.size() && v[i] == ':') {
        i = skip_ws(v, i + 1);
        size_t j = i;
        while (j < v.size() && !is_space(v[j])) ++j;
        if (j > i && skip_ws(v, j) == v.size()) {
          *nb = i;
          *ne = j;
          return true;
        }
      }
    }
  }
  // ^\s*\.section\s+\.text\.([^,\s]+)
  {
    size_t i = skip_ws(v, 0);
    View w{v.p, v.b + i, v.e};
    if (starts_with(w, ".section")) {
      size_t j = skip_ws(v, i + 8);
      if (j > i + 8) {
        View x{v.p, v.b + j, v.e};
        if (starts_with(x, ".text.")) {
          size_t s = j + 6, t = s;
          while (t < v.size() && v[t] != ',' && !is_space(v[t])) ++t;
          if (t > s) {
            *nb = s;
            *ne = t;
            return true;
          }
        }
      }
    }
  }
  return label_match(v, nb, ne);
}

// ^([A-Z][A-Z0-9]*)((?:\.[^\s.]+)*)$ ; op_end = end of group 1
bool opcode_match(View v, size_t* op_end) {
  if (v.empty() || !is_upper(v[0])) return false;
  size_t i = 1;
  while (i < v.size() && is_upper_digit(v[i])) ++i;
  *op_end = i;
  while (i < v.size()) {
    if (v[i] != '.') return false;
    size_t j = i + 1;
    while (j < v.size() && v[j] != '.' && !is_space(v[j])) ++j;
    if (j == i + 1) return false;
    i = j;
  }
  return true;
}

// count of \bR\d+\b matches in a token (findall, non-overlapping)
uint32_t count_regs(View t) {
  uint32_t n = 0;
  size_t p = 0;
  while (p < t.size()) {
    if (t[p] == 'R' && (p == 0 || !is_word(t[p - 1]))) {
      size_t q = p + 1;
      while (q < t.size() && is_digit(t[q])) ++q;
      if (q > p + 1 && (q == t.size() || !is_word(t[q]))) {
        ++n;
        p = q;
        continue;
      }
    }
    ++p;
  }
  return n;
}

enum { kNone = 0, kInstr = 1, kErrGuard = 2, kErrSemicolon = 3, kErrAttr = 4 };

struct ParsedInstr {
  std::string sig;       // opcode \x1f .mod \x1f .mod ...
  bool guard;
  uint32_t regops;
  std::string token;     // opcode token for the ';' error message
};

void append_utf8(std::string& s, uint32_t c) {
  if (c < 0x80) s.push_back((char)c);
  else if (c < 0x800) {
    s.push_back((char)(0xC0 | (c >> 6)));
    s.push_back((char)(0x80 | (c & 0x3F)));
  } else if (c < 0x10000) {
    s.push_back((char)(0xE0 | (c >> 12)));
    s.push_back((char)(0x80 | ((c >> 6) & 0x3F)));
    s.push_back((char)(0x80 | (c & 0x3F)));
  } else {
    s.push_back((char)(0xF0 | (c >> 18)));
    s.push_back((char)(0x80 | ((c >> 12) & 0x3F)));
    s.push_back((char)(0x80 | ((c >> 6) & 0x3F)));
    s.push_back((char)(0x80 | (c & 0x3F)));
  }
}
std::string to_utf8(View v) {
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) append_utf8(s, v[i]);
  return s;
}

// parse_instruction_line (sass.py:236-288)
int parse_instruction(View line, ParsedInstr& out) {
  // scheduling-control prefix ^\s*\[[-\w:]+\]  (one substitution)
  {
    size_t i = skip_ws(line, 0);
    if (i < line.size() && line[i] == '[') {
      size_t j = i + 1;
      while (j < line.size() && (line[j] == '-' || line[j] == ':' || is_word(line[j]))) ++j;
      if (j > i + 1 && j < line.size() && line[j] == ']') line.b += j + 1;
    }
  }
  // address ^\s*/\*\s*([0-9a-fA-F]+)\s*\*/
  {
    size_t i = skip_ws(line, 0);
    if (i + 1 < line.size() && line[i] == '/' && line[i + 1] == '*') {
      size_t j = skip_ws(line, i + 2), k = j;
      while (k < line.size() && is_hex(line[k])) ++k;
      if (k > j) {
        size_t m = skip_ws(line, k);
        if (m + 1 < line.size() && line[m] == '*' && line[m + 1] == '/') line.b += m + 2;
      }
    }
  }
  // trailing comments: /\*.*?\*/\s*$ removed repeatedly, rstrip each round
  for (;;) {
    const size_t before_b = line.b, before_e = line.e;
    // the only "*/" that can be followed by whitespace to the end is the last one
    size_t J = (size_t)-1;
    for (size_t j = line.size(); j-- > 1;)
      if (line[j - 1] == '*' && line[j] == '/') {
        J = j - 1;
        break;
      }
    if (J != (size_t)-1 && skip_ws(line, J + 2) == line.size()) {
      for (size_t i = 0; i + 2 <= J && i + 1 < line.size(); ++i)
        if (line[i] == '/' && line[i + 1] == '*') {
          line.e = line.b + i;
          break;
        }
    }
    line = rstrip(line);
    if (line.b == before_b && line.e == before_e) break;
  }
  line = strip(line);
  while (!line.empty() && (line[0] == '{' || line[0] == '}')) ++line.b;
  while (!line.empty() && (line[line.size() - 1] == '{' || line[line.size() - 1] == '}')) --line.e;
  line = strip(line);
  if (line.empty() || starts_with(line, ".") || starts_with(line, "//")) return kNone;
  if (starts_with(line, "/*")) return kNone;
  if (label_match(line, nullptr, nullptr)) return kNone;

  // predicate guard: body.partition(" ")
  View body = line;
  out.guard = false;
  {
    size_t sp = 0;
    while (sp < line.size() && line[sp] != ' ') ++sp;
    View first{line.p, line.b, line.b + sp};
    // ^@!?P\w+$  (the |^@!?PT$ alternative is a subset)
    bool pred = false;
    if (first.size() >= 3 && first[0] == '@') {
      size_t i = 1;
      if (first[i] == '!') ++i;
      if (i < first.size() && first[i] == 'P') {
        ++i;
        if (i < first.size()) {
          pred = true;
          for (size_t k = i; k < first.size(); ++k)
            if (!is_word(first[k])) {
              pred = false;
              break;
            }
        }
      }
    }
    if (pred) {
      out.guard = true;
      View rest{line.p, sp < line.size() ? line.b + sp + 1 : line.e, line.e};
      body = strip(rest);
      if (body.empty()) return kErrGuard;
    }
  }
  // opcode_token = body.split(None, 1)[0].rstrip(";")
  View tok = body;
  {
    size_t i = 0;
    while (i < tok.size() && !is_space(tok[i])) ++i;
    tok.e = tok.b + i;
    while (!tok.empty() && tok[tok.size() - 1] == ';') --tok.e;
  }
  size_t op_end = 0;
  if (!opcode_match(tok, &op_end)) return kNone;
  View br = rstrip(body);
  if (br.empty() || br[br.size() - 1] != ';') {
    out.token = to_utf8(tok);
    return kErrSemicolon;
  }
  br.e -= 1;
  View b2 = strip(br);
  size_t sp = 0;
  while (sp < b2.size() && b2[sp] != ' ') ++sp;
  View head{b2.p, b2.b, b2.b + sp};
  View operands{b2.p, sp < b2.size() ? b2.b + sp + 1 : b2.e, b2.e};
  if (!opcode_match(head, &op_end)) return kErrAttr;   // sass.py:279 m.group on None
  std::string sig;
  for (size_t i = 0; i < op_end; ++i) sig.push_back((char)head[i]);
  {
    size_t i = op_end;
    while (i < head.size()) {                            // group 2: (\.[^\s.]+)*
      size_t j = i + 1;
      while (j < head.size() && head[j] != '.') ++j;
      sig.push_back('\x1f');
      View part{head.p, head.b + i + 1, head.b + j};     // without the dot
      sig += to_utf8(part);
      i = j;
    }
  }
  // operands: text.split(",") -> strip -> non-empty
  uint32_t regs = 0;
  {
    size_t s = 0;
    for (size_t i = 0; i <= operands.size(); ++i) {
      if (i == operands.size() || operands[i] == ',') {
        View t = strip(View{operands.p, operands.b + s, operands.b + i});
        if (!t.empty()) regs += count_regs(t);
        s = i + 1;
      }
    }
  }
  out.sig = std::move(sig);
  out.regops = regs;
  return kInstr;
}

// decode UTF-8 (incl. surrogate code points, as produced by 'surrogatepass')
inline uint32_t next_cp(const unsigned char* s, size_t n, size_t& i) {
  const unsigned char c = s[i];
  if (c < 0x80) {
    ++i;
    return c;
  }
  if ((c >> 5) == 6 && i + 1 < n) {
    const uint32_t v = ((c & 0x1F) << 6) | (s[i + 1] & 0x3F);
    i += 2;
    return v;
  }
  if ((c >> 4) == 14 && i + 2 < n) {
    const uint32_t v = ((c & 0x0F) << 12) | ((s[i + 1] & 0x3F) << 6) | (s[i + 2] & 0x3F);
    i += 3;
    return v;
  }
  if ((c >> 3) == 30 && i + 3 < n) {
    const uint32_t v = ((c & 0x07) << 18) | ((s[i + 1] & 0x3F) << 12) |
                       ((s[i + 2] & 0x3F) << 6) | (s[i + 3] & 0x3F);
    i += 4;
    return v;
  }
  ++i;
  return 0xFFFD;
}

inline bool is_linebreak(uint32_t c) {
  return (c >= 0x0A && c <= 0x0D) || (c >= 0x1C && c <= 0x1E) || c == 0x85 || c == 0x2028 ||
         c == 0x2029;
}

// ---------------------------------------------------------------------------
// Chunked parse.  The text is cut after '\n' bytes into line-aligned chunks
// parsed concurrently; each chunk records its function starts, instructions
// (with chunk-local signature ids) and its first error, then the chunks are
// merged in order.  Instructions before a chunk's first header belong to the
// function still open at the end of the previous chunk, so "instruction
// before any function header" is only decided in the merge.
// ---------------------------------------------------------------------------
struct FnStart {
  std::string name;
  uint64_t at;            // chunk-local instruction index where it starts
};

struct Chunk {
  uint64_t lines = 0;
  bool any_header = false;
  std::vector<FnStart> fns;
  std::vector<uint32_t> recs;            // local signature ids
  std::vector<std::string> sigs;
  std::unordered_map<std::string, uint32_t> sig_ids;
  uint64_t first_instr_line = 0;         // line of the first instruction before a header
  int err = 0;                           // kErr* of the first line-local error
  uint64_t err_line = 0;                 // chunk-local 1-based
  std::string err_text;
};

void parse_chunk(const unsigned char* s, size_t n, Chunk& ck) {
  Str line;
  line.reserve(512);
  ParsedInstr pi;
  pi.sig.reserve(64);
  size_t i = 0;
  bool seen_header = false;
  while (i < n) {
    line.clear();
    while (i < n) {
      const unsigned char b = s[i];
      uint32_t c;
      if (b < 0x80) {                       // ASCII fast path
        ++i;
        if (b == '\n' || b == '\r' || b == 0x0B || b == 0x0C || (b >= 0x1C && b <= 0x1E)) {
          if (b == '\r' && i < n && s[i] == '\n') ++i;
          goto line_done;
        }
        line.push_back(b);
        continue;
      }
      c = next_cp(s, n, i);
      if (c == 0x85 || c == 0x2028 || c == 0x2029) goto line_done;
      line.push_back(c);
    }
  line_done:
    ++ck.lines;
    View v{line.data(), 0, line.size()};
    size_t nb = 0, ne = 0;
    if (header_name(v, &nb, &ne)) {
      ck.any_header = true;
      if (ck.err) break;                   // error fixed; EmptyInput ruled out
      seen_header = true;
      ck.fns.push_back(FnStart{to_utf8(View{line.data(), nb, ne}), ck.recs.size()});
      continue;
    }
    if (ck.err) continue;
    const int k = parse_instruction(v, pi);
    if (k == kNone) continue;
    if (k == kErrGuard || k == kErrSemicolon || k == kErrAttr) {
      ck.err = k;
      ck.err_line = ck.lines;
      ck.err_text = k == kErrSemicolon ? std::string("\x01") + pi.token : std::string();
      continue;
    }
    if (!seen_header && ck.recs.empty()) ck.first_instr_line = ck.lines;
    if (pi.regops > 255) {
      ck.err = 5;
      ck.err_line = ck.lines;
      continue;
    }
    auto it = ck.sig_ids.find(pi.sig);
    uint32_t id;
    if (it == ck.sig_ids.end()) {
      id = (uint32_t)ck.sigs.size();
      ck.sig_ids.emplace(pi.sig, id);
      ck.sigs.push_back(pi.sig);
    } else {
      id = it->second;
    }
    ck.recs.push_back(OCCX_INSTR(id, pi.regops, pi.guard ? 1u : 0u));
  }
}

}  // namespace

struct occx_sass {
  std::vector<std::string> names;
  std::vector<uint64_t> offsets;   // n_kernels + 1
  std::vector<uint32_t> records;
  std::vector<std::string> sigs;
  std::string error;               // message (';' error: 0x01 + offending token)
  int64_t error_line = 0;
  std::string names_blob, sigs_blob;   // all names / signatures joined by 0x1E
};

extern "C" int occx_sass_parse(const char* text, uint64_t n_bytes, occx_sass** out,
                               int64_t* err_line) {
  return occx_sass_parse_ex(text, n_bytes, 0, out, err_line);
}

extern "C" int occx_sass_parse_ex(const char* text, uint64_t n_bytes, uint64_t chunk_bytes_min,
                                  occx_sass** out, int64_t* err_line) {
  if (!out) return OCCX_ERR_VALUE;
  occx_sass* r = new occx_sass();
  *out = r;
  if (err_line) *err_line = 0;
  const unsigned char* s = reinterpret_cast<const unsigned char*>(text);
  // line-aligned chunks (cut after '\n'; a "\r\n" pair never straddles a cut)
  unsigned hw = std::thread::hardware_concurrency();
  const unsigned max_t = hw ? (hw < 32 ? hw : 32) : 1;
  // >= 1 MB per chunk by default (every core on mid-size listings); callers
  // (tests) may force small chunks
  const uint64_t chunk_bytes = chunk_bytes_min ? chunk_bytes_min : (uint64_t)(1u << 20);
  unsigned n_chunks = (unsigned)(n_bytes / chunk_bytes) + 1;
  if (n_chunks > max_t) n_chunks = max_t;
  std::vector<size_t> cut{0};
  for (unsigned c = 1; c < n_chunks; ++c) {
    size_t p = (size_t)((n_bytes * (uint64_t)c) / n_chunks);
    if (p <= cut.back()) continue;
    while (p < n_bytes && s[p - 1] != '\n') ++p;
    if (p < n_bytes) cut.push_back(p);
  }
  cut.push_back(n_bytes);
  std::vector<Chunk> ck(cut.size() - 1);
  if (ck.size() == 1) {
    parse_chunk(s, n_bytes, ck[0]);
  } else {
    std::vector<std::thread> th;
    for (size_t c = 0; c < ck.size(); ++c)
      th.emplace_back(parse_chunk, s + cut[c], cut[c + 1] - cut[c], std::ref(ck[c]));
    for (auto& t : th) t.join();
  }
  // merge in order
  bool any_header = false;
  for (auto& c : ck) any_header |= c.any_header;
  if (!any_header) {
    r->error = "no functions found";
    return OCCX_ERR_EMPTY;
  }
  // Global signature ids in first-occurrence order, without a serial pass
  // over every chunk's table: partition p of P (by hash) walks the chunks in
  // order and records, for each local signature of its partition, the
  // (chunk, local index) of the signature's first occurrence -- its "owner".
  // The serial pass below then numbers the owners in chunk order.
  const size_t C = ck.size();
  std::vector<std::vector<uint64_t>> owner(C);
  std::vector<std::vector<size_t>> hashes(C);
  {
    auto hash_chunk = [&](size_t ci) {
      hashes[ci].resize(ck[ci].sigs.size());
      owner[ci].resize(ck[ci].sigs.size());
      for (size_t i = 0; i < ck[ci].sigs.size(); ++i)
        hashes[ci][i] = std::hash<std::string>{}(ck[ci].sigs[i]);
    };
    const unsigned P = C > 1 ? (unsigned)C : 1u;
    auto partition = [&](unsigned part) {
      std::unordered_map<std::string_view, uint64_t> first;
      for (size_t ci = 0; ci < C; ++ci)
        for (size_t i = 0; i < ck[ci].sigs.size(); ++i) {
          if (hashes[ci][i] % P != part) continue;
          const uint64_t key = ((uint64_t)ci << 32) | i;
          owner[ci][i] = first.emplace(std::string_view(ck[ci].sigs[i]), key).first->second;
        }
    };
    if (C == 1) {
      hash_chunk(0);
      partition(0);
    } else {
      std::vector<std::thread> th;
      for (size_t ci = 0; ci < C; ++ci) th.emplace_back(hash_chunk, ci);
      for (auto& t : th) t.join();
      th.clear();
      for (unsigned part = 0; part < P; ++part) th.emplace_back(partition, part);
      for (auto& t : th) t.join();
    }
  }
  // serial pass: global signature ids, function starts (as output positions)
  // and errors in chunk order; the records are copied afterwards, one thread
  // per chunk
  std::vector<std::vector<uint32_t>> remaps(ck.size());
  std::vector<uint64_t> rec_base(ck.size() + 1, 0);
  bool have_fn = false;
  std::string cur;
  uint64_t line_base = 0;
  auto fail = [&](int status, uint64_t line, std::string msg) {
    r->error = std::move(msg);
    r->error_line = (int64_t)line;
    if (err_line) *err_line = (int64_t)line;
    return status;
  };
  for (size_t ci = 0; ci < ck.size(); ++ci) {
    Chunk& c = ck[ci];
    // instructions before this chunk's first header continue the open function
    const uint64_t lead = c.fns.empty() ? c.recs.size() : c.fns[0].at;
    if (lead > 0 && !have_fn)
      return fail(OCCX_ERR_PARSE, line_base + c.first_instr_line,
                  "instruction before any function header");
    std::vector<uint32_t>& remap = remaps[ci];
    remap.resize(c.sigs.size());
    for (size_t i = 0; i < c.sigs.size(); ++i) {
      const uint64_t o = owner[ci][i];
      const size_t oc = (size_t)(o >> 32), oi = (size_t)(o & 0xffffffffu);
      if (oc == ci && oi == i) {                            // first occurrence: a new id
        const uint32_t id = (uint32_t)r->sigs.size();
        if (id >= 65535)
          return fail(OCCX_ERR_CAPACITY, line_base + 1,
                      "more than 65535 distinct instruction signatures");
        r->sigs.push_back(c.sigs[i]);
        remap[i] = id;
      } else {
        remap[i] = remaps[oc][oi];                          // an earlier chunk (or index)
      }
    }
    for (const FnStart& fs : c.fns) {
      if (!have_fn || fs.name != cur) {
        if (have_fn) r->offsets.push_back(rec_base[ci] + fs.at);
        r->names.push_back(fs.name);
        cur = fs.name;
        have_fn = true;
      }
    }
    if (c.err) {
      const uint64_t line = line_base + c.err_line;
      if (c.err == kErrGuard) return fail(OCCX_ERR_PARSE, line, "predicate guard with no instruction");
      if (c.err == kErrSemicolon) return fail(OCCX_ERR_PARSE, line, c.err_text);
      if (c.err == kErrAttr)
        return fail(OCCX_ERR_ATTRIBUTE, line, "'NoneType' object has no attribute 'group'");
      return fail(OCCX_ERR_CAPACITY, line, "instruction with more than 255 register operands");
    }
    rec_base[ci + 1] = rec_base[ci] + c.recs.size();
    line_base += c.lines;
  }
  r->records.resize(rec_base.back());
  auto fill = [&](size_t ci) {
    const std::vector<uint32_t>& remap = remaps[ci];
    uint32_t* dst = r->records.data() + rec_base[ci];
    for (const uint32_t x : ck[ci].recs) *dst++ = (remap[(x >> 1) & 0xffffu] << 1) | (x & 0xfffe0001u);
  };
  if (ck.size() == 1) {
    fill(0);
  } else {
    std::vector<std::thread> th;
    for (size_t ci = 0; ci < ck.size(); ++ci) th.emplace_back(fill, ci);
    for (auto& t : th) t.join();
  }
  if (have_fn) r->offsets.push_back(r->records.size());
  r->offsets.insert(r->offsets.begin(), 0);
  // one-call views of the names and signatures (0x1E is a line break, so it
  // occurs in neither)
  for (size_t i = 0; i < r->names.size(); ++i) {
    if (i) r->names_blob.push_back('\x1e');
    r->names_blob += r->names[i];
  }
  for (size_t i = 0; i < r->sigs.size(); ++i) {
    if (i) r->sigs_blob.push_back('\x1e');
    r->sigs_blob += r->sigs[i];
  }
  return OCCX_OK;
}

extern "C" uint32_t occx_sass_n_kernels(const occx_sass* r) { return r ? (uint32_t)r->names.size() : 0; }
extern "C" uint64_t occx_sass_n_instr(const occx_sass* r) { return r ? r->records.size() : 0; }
extern "C" const uint32_t* occx_sass_records(const occx_sass* r) {
  return r && !r->records.empty() ? r->records.data() : nullptr;
}
extern "C" const uint64_t* occx_sass_offsets(const occx_sass* r) {
  return r && !r->offsets.empty() ? r->offsets.data() : nullptr;
}
extern "C" const char* occx_sass_kernel_name(const occx_sass* r, uint32_t k) {
  return r && k < r->names.size() ? r->names[k].c_str() : nullptr;
}
extern "C" uint32_t occx_sass_n_sigs(const occx_sass* r) { return r ? (uint32_t)r->sigs.size() : 0; }
extern "C" const char* occx_sass_signature(const occx_sass* r, uint32_t i) {
  return r && i < r->sigs.size() ? r->sigs[i].c_str() : nullptr;
}
extern "C" const char* occx_sass_error_text(const occx_sass* r) { return r ? r->error.c_str() : ""; }
extern "C" const char* occx_sass_names_blob(const occx_sass* r, uint64_t* n_bytes) {
  if (n_bytes) *n_bytes = r ? r->names_blob.size() : 0;
  return r ? r->names_blob.c_str() : "";
}
extern "C" const char* occx_sass_signatures_blob(const occx_sass* r, uint64_t* n_bytes) {
  if (n_bytes) *n_bytes = r ? r->sigs_blob.size() : 0;
  return r ? r->sigs_blob.c_str() : "";
}

// Replace every record's signature id by its class id (sig_class[sig],
// classify() of the interned signature, mix.py:176-187): "class records",
// reduced by K0 with the identity class table (n_sig = 15), whose lookups
// are conflict-free in shared memory.  Threaded over record ranges.
extern "C" int occx_sass_classify(occx_sass* r, const uint8_t* sig_class, uint32_t n_sig) {
  if (!r || !sig_class || n_sig < r->sigs.size()) return OCCX_ERR_VALUE;
  for (uint32_t i = 0; i < (uint32_t)r->sigs.size(); ++i)
    if (sig_class[i] > 14) return OCCX_ERR_VALUE;
  const size_t n = r->records.size();
  uint32_t* rec = r->records.data();
  auto run = [&](size_t b, size_t e) {
    for (size_t i = b; i < e; ++i) {
      const uint32_t x = rec[i];
      rec[i] = (x & 0xfffe0001u) | ((uint32_t)sig_class[(x >> 1) & 0xffffu] << 1);
    }
  };
  unsigned hw = std::thread::hardware_concurrency();
  const size_t nt = std::min<size_t>(hw ? (hw < 32 ? hw : 32) : 1, n / (1u << 20) + 1);
  if (nt <= 1) {
    run(0, n);
  } else {
    std::vector<std::thread> th;
    for (size_t t = 0; t < nt; ++t) th.emplace_back(run, n * t / nt, n * (t + 1) / nt);
    for (auto& t : th) t.join();
  }
  return OCCX_OK;
}
extern "C" void occx_sass_free(occx_sass* r) { delete r; }
