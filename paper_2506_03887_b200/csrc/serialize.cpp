// serialize.cpp — the reference's on-disk formats:
//
//   GMASKDP1   SerializeDpda / DeserializeDpda (src/serialize.cpp:148-294):
//              "GMASKDP1\n" + one JSON object, keys sorted, compact, "\n".
//              The writer reproduces the reference's bytes exactly (its JSON
//              library dumps std::map-ordered keys without whitespace); the
//              loader re-derives arbitration order and re-checks determinism
//              (serialize.cpp:284-292), so a tampered file cannot smuggle in an
//              inconsistent machine.
//   vocabulary LoadVocabulary (serialize.cpp:348-364): a JSON array of
//              strings whose entries are then `\xNN` / `\\` unescaped
//              (UnescapeToken, :315-346); EscapeToken (:298-313) inverts it.
//
// The JSON reader/writer below is this file's own minimal implementation of
// exactly what these formats use (objects, arrays, strings, integers,
// booleans); errors map to GM_ERR_CORRUPT_INPUT with the reference's
// SerializeError kinds in the message (BadMagic / BadVersion / Parse /
// Structure).
#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "gm_internal.hpp"

namespace pre3 {
namespace {

constexpr char kDp1Magic[] = "GMASKDP1";

[[noreturn]] void Bad(const char* kind, const std::string& msg) {
  throw Error(GM_ERR_CORRUPT_INPUT, std::string("SerializeError(") + kind + "): " + msg);
}

// ---------------------------------------------------------------- writer
void PutStr(std::string* o, const std::string& s) {
  o->push_back('"');
  for (unsigned char c : s) {
    switch (c) {
      case '"': *o += "\\\""; break;
      case '\\': *o += "\\\\"; break;
      case '\b': *o += "\\b"; break;
      case '\f': *o += "\\f"; break;
      case '\n': *o += "\\n"; break;
      case '\r': *o += "\\r"; break;
      case '\t': *o += "\\t"; break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", c);
          *o += buf;
        } else {
          o->push_back(static_cast<char>(c));
        }
    }
  }
  o->push_back('"');
}

void PutInts(std::string* o, const std::vector<int32_t>& v) {
  o->push_back('[');
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) o->push_back(',');
    *o += std::to_string(v[i]);
  }
  o->push_back(']');
}

// ByteSet::ToHex (grammar.cpp:324-331): 64 hex digits, low nibble of word 0 first.
std::string HexOf(const uint64_t w[4]) {
  static const char* d = "0123456789abcdef";
  std::string out(64, '0');
  for (int i = 0; i < 64; ++i) out[static_cast<size_t>(i)] = d[(w[i / 16] >> ((i % 16) * 4)) & 0xf];
  return out;
}

// One edge object, keys in sorted order.
void PutEdge(std::string* o, const Edge& e, bool composite) {
  *o += "{\"accepted\":";
  PutStr(o, HexOf(e.accepted));
  *o += ",\"dollar\":";
  *o += e.dollar ? "true" : "false";
  *o += ",\"dynamic\":";
  *o += e.dynamic ? "true" : "false";
  *o += ",\"match\":";
  PutInts(o, e.match_pop);
  *o += ",\"origin\":" + std::to_string(e.origin);
  *o += ",\"push\":";
  PutInts(o, e.push);
  if (composite) {
    *o += ",\"second\":";
    PutStr(o, HexOf(e.second));
    *o += ",\"second_dollar\":";
    *o += e.dollar_second ? "true" : "false";
  }
  *o += ",\"source\":" + std::to_string(e.source);
  *o += ",\"target\":" + std::to_string(e.target) + "}";
}

// ---------------------------------------------------------------- reader
struct JVal {
  enum Kind { kNull, kBool, kInt, kFloat, kStr, kArr, kObj } kind = kNull;
  bool b = false;
  int64_t i = 0;
  std::string s;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
};

struct JParser {
  const char* p;
  const char* end;
  int depth = 0;

  [[noreturn]] void Fail(const std::string& m) { Bad("Parse", m); }
  void Ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool Lit(const char* w) {
    const size_t n = std::strlen(w);
    if (static_cast<size_t>(end - p) >= n && std::memcmp(p, w, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  static void Utf8(std::string* o, uint32_t cp) {
    if (cp < 0x80) {
      o->push_back(static_cast<char>(cp));
    } else if (cp < 0x800) {
      o->push_back(static_cast<char>(0xC0 | (cp >> 6)));
      o->push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
      o->push_back(static_cast<char>(0xE0 | (cp >> 12)));
      o->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      o->push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else {
      o->push_back(static_cast<char>(0xF0 | (cp >> 18)));
      o->push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
      o->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      o->push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    }
  }
  uint32_t Hex4() {
    if (end - p < 4) Fail("truncated \\u escape");
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
      else Fail("bad \\u escape");
    }
    return v;
  }
  std::string Str() {
    ++p;  // opening quote
    std::string o;
    for (;;) {
      if (p >= end) Fail("unterminated string");
      const unsigned char c = static_cast<unsigned char>(*p++);
      if (c == '"') return o;
      if (c < 0x20) Fail("control character in string");
      if (c != '\\') {
        o.push_back(static_cast<char>(c));
        continue;
      }
      if (p >= end) Fail("dangling escape");
      const char e = *p++;
      switch (e) {
        case '"': o.push_back('"'); break;
        case '\\': o.push_back('\\'); break;
        case '/': o.push_back('/'); break;
        case 'b': o.push_back('\b'); break;
        case 'f': o.push_back('\f'); break;
        case 'n': o.push_back('\n'); break;
        case 'r': o.push_back('\r'); break;
        case 't': o.push_back('\t'); break;
        case 'u': {
          uint32_t cp = Hex4();
          if (cp >= 0xD800 && cp < 0xDC00) {  // surrogate pair
            if (!Lit("\\u")) Fail("unpaired surrogate");
            const uint32_t lo = Hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) Fail("bad surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp < 0xE000) {
            Fail("unpaired surrogate");
          }
          Utf8(&o, cp);
          break;
        }
        default: Fail(std::string("bad escape \\") + e);
      }
    }
  }
  JVal Val() {
    if (++depth > 64) Fail("nesting too deep");
    Ws();
    if (p >= end) Fail("unexpected end of input");
    JVal v;
    const char c = *p;
    if (c == '{') {
      ++p;
      v.kind = JVal::kObj;
      Ws();
      if (p < end && *p == '}') {
        ++p;
      } else {
        for (;;) {
          Ws();
          if (p >= end || *p != '"') Fail("expected object key");
          std::string k = Str();
          Ws();
          if (p >= end || *p != ':') Fail("expected ':'");
          ++p;
          v.obj[k] = Val();
          Ws();
          if (p < end && *p == ',') {
            ++p;
            continue;
          }
          if (p < end && *p == '}') {
            ++p;
            break;
          }
          Fail("expected ',' or '}'");
        }
      }
    } else if (c == '[') {
      ++p;
      v.kind = JVal::kArr;
      Ws();
      if (p < end && *p == ']') {
        ++p;
      } else {
        for (;;) {
          v.arr.push_back(Val());
          Ws();
          if (p < end && *p == ',') {
            ++p;
            continue;
          }
          if (p < end && *p == ']') {
            ++p;
            break;
          }
          Fail("expected ',' or ']'");
        }
      }
    } else if (c == '"') {
      v.kind = JVal::kStr;
      v.s = Str();
    } else if (Lit("true")) {
      v.kind = JVal::kBool;
      v.b = true;
    } else if (Lit("false")) {
      v.kind = JVal::kBool;
    } else if (Lit("null")) {
      v.kind = JVal::kNull;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      const char* q = p;
      if (*q == '-') ++q;
      if (q >= end || *q < '0' || *q > '9') Fail("bad number");
      while (q < end && *q >= '0' && *q <= '9') ++q;
      bool is_float = false;
      if (q < end && *q == '.') {
        is_float = true;
        ++q;
        while (q < end && *q >= '0' && *q <= '9') ++q;
      }
      if (q < end && (*q == 'e' || *q == 'E')) {
        is_float = true;
        ++q;
        if (q < end && (*q == '+' || *q == '-')) ++q;
        while (q < end && *q >= '0' && *q <= '9') ++q;
      }
      const std::string num(p, q);
      p = q;
      if (is_float) {
        v.kind = JVal::kFloat;
      } else {
        v.kind = JVal::kInt;
        errno = 0;
        char* stop = nullptr;
        v.i = std::strtoll(num.c_str(), &stop, 10);
        if (errno != 0) v.kind = JVal::kFloat;  // out of int64 range: not an integer field
      }
    } else {
      Fail(std::string("unexpected character '") + c + "'");
    }
    --depth;
    return v;
  }
};

JVal ParseJson(const char* p, const char* end) {
  JParser ps{p, end};
  JVal v = ps.Val();
  ps.Ws();
  if (ps.p != end) Bad("Parse", "trailing characters after JSON value");
  return v;
}

// Field accessors with the reference's structure errors (serialize.cpp:46-105).
const JVal& Field(const JVal& j, const char* k) {
  auto it = j.obj.find(k);
  if (it == j.obj.end()) Bad("Structure", std::string("missing field ") + k);
  return it->second;
}
int64_t IntField(const JVal& j, const char* k) {
  const JVal& f = Field(j, k);
  if (f.kind != JVal::kInt) Bad("Structure", std::string("field ") + k + " must be an integer");
  return f.i;
}
std::string StrField(const JVal& j, const char* k) {
  const JVal& f = Field(j, k);
  if (f.kind != JVal::kStr) Bad("Structure", std::string("field ") + k + " must be a string");
  return f.s;
}
bool BoolField(const JVal& j, const char* k) {
  const JVal& f = Field(j, k);
  if (f.kind != JVal::kBool) Bad("Structure", std::string("field ") + k + " must be a boolean");
  return f.b;
}
std::vector<int32_t> StateVec(const JVal& j, const char* k, int64_t num_states) {
  const JVal& f = Field(j, k);
  if (f.kind != JVal::kArr) Bad("Structure", std::string("field ") + k + " must be an array");
  std::vector<int32_t> out;
  for (const JVal& v : f.arr) {
    if (v.kind != JVal::kInt) Bad("Structure", std::string(k) + " entries must be integers");
    if (v.i < 0 || v.i >= num_states) {
      Bad("Structure", std::string(k) + " entry " + std::to_string(v.i) + " out of range");
    }
    out.push_back(static_cast<int32_t>(v.i));
  }
  return out;
}
void HexField(const JVal& j, const char* k, uint64_t w[4]) {
  const std::string h = StrField(j, k);
  if (h.size() != 64) Bad("Structure", std::string(k) + ": byte set hex must be 64 chars");
  w[0] = w[1] = w[2] = w[3] = 0;
  for (int i = 0; i < 64; ++i) {
    const char c = h[static_cast<size_t>(i)];
    int v = -1;
    if (c >= '0' && c <= '9') v = c - '0';
    else if (c >= 'a' && c <= 'f') v = c - 'a' + 10;
    else if (c >= 'A' && c <= 'F') v = c - 'A' + 10;
    if (v < 0) Bad("Structure", std::string(k) + ": bad hex digit in byte set");
    w[i / 16] |= static_cast<uint64_t>(v) << ((i % 16) * 4);
  }
}

// EdgeFromJson (serialize.cpp:107-144).
Edge EdgeOf(const JVal& j, int64_t S, bool composite) {
  Edge e;
  const int64_t source = IntField(j, "source");
  if (source < 0 || source >= S) Bad("Structure", "edge source out of range");
  e.source = static_cast<int32_t>(source);
  HexField(j, "accepted", e.accepted);
  e.dollar = BoolField(j, "dollar");
  e.dynamic = BoolField(j, "dynamic");
  e.match_pop = StateVec(j, "match", S);
  e.push = StateVec(j, "push", S);
  const int64_t origin = IntField(j, "origin");
  if (origin < 0 || origin > 3) Bad("Structure", "edge origin out of range");
  e.origin = static_cast<uint8_t>(origin);
  const int64_t target = IntField(j, "target");
  if (target < -1 || target >= S) Bad("Structure", "edge target out of range");
  e.target = static_cast<int32_t>(target);
  if (e.match_pop.empty() || e.match_pop.front() != e.source) {
    Bad("Structure", "edge condition must start at its source state");
  }
  if (e.dynamic) {
    if (e.target != -1 || e.push.empty() || e.dollar) Bad("Structure", "dynamic edge shape is inconsistent");
  } else if (e.target == -1) {
    Bad("Structure", "static edge lacks a target");
  }
  if (composite) {
    HexField(j, "second", e.second);
    e.dollar_second = BoolField(j, "second_dollar");
  }
  return e;
}

std::string HashHex(uint64_t h) {
  char buf[17];
  std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(h));
  return buf;
}

}  // namespace

std::vector<uint8_t> SaveGmaskdp1(const Automaton& a) {
  std::string o = std::string(kDp1Magic) + "\n";
  o += "{\"accept_state\":" + std::to_string(a.accept_state);
  o += ",\"composites\":[";
  for (size_t i = 0; i < a.composite_edges.size(); ++i) {
    if (i) o.push_back(',');
    PutEdge(&o, a.composite_edges[i], true);
  }
  o += "],\"cycles\":[";
  for (size_t i = 0; i < a.cycle_list.size(); ++i) {
    if (i) o.push_back(',');
    o += "{\"closing_byte\":" + std::to_string(a.cycle_list[i].closing_byte) + ",\"states\":";
    PutInts(&o, a.cycle_list[i].states);
    o.push_back('}');
  }
  o += "],\"edges\":[";
  for (size_t i = 0; i < a.edges.size(); ++i) {
    if (i) o.push_back(',');
    PutEdge(&o, a.edges[i], false);
  }
  o += "],\"grammar_hash\":";
  PutStr(&o, HashHex(a.grammar_hash));
  o += ",\"grammar_text\":";
  PutStr(&o, a.grammar_text);
  o += ",\"initial_state\":" + std::to_string(a.initial_state);
  o += ",\"num_states\":" + std::to_string(a.num_states);
  o += ",\"shifts\":[";
  bool first = true;
  for (int32_t s = 0; s < a.num_states; ++s) {
    for (int b = 0; b < 256; ++b) {
      const int32_t t = a.shift_targets[static_cast<size_t>(s) * 256 + static_cast<size_t>(b)];
      if (t < 0) continue;
      if (!first) o.push_back(',');
      first = false;
      o += "[" + std::to_string(s) + "," + std::to_string(b) + "," + std::to_string(t) + "]";
    }
  }
  const BuildStats& st = a.stats;
  o += "],\"stats\":{\"acceptance_edges\":" + std::to_string(st.acceptance) +
       ",\"aggregated_groups\":" + std::to_string(st.aggregated_groups) +
       ",\"cycle_back_edges\":" + std::to_string(st.cycle_back) +
       ",\"edges_before_aggregation\":" + std::to_string(st.edges_before_aggregation) +
       ",\"merged_edges\":" + std::to_string(st.merged) + ",\"reduction_edges\":" + std::to_string(st.reduction) +
       ",\"states\":" + std::to_string(st.states) + "},\"version\":1}\n";
  return std::vector<uint8_t>(o.begin(), o.end());
}

// DeserializeDpda (serialize.cpp:198-294).
Automaton LoadGmaskdp1(const uint8_t* data, size_t n) {
  const char* p = reinterpret_cast<const char*>(data);
  const char* nl = static_cast<const char*>(std::memchr(p, '\n', n));
  if (nl == nullptr || std::string(p, nl) != kDp1Magic) Bad("BadMagic", "missing or wrong magic line");
  JVal j;
  try {
    j = ParseJson(nl + 1, p + n);
  } catch (const Error&) {
    Bad("Parse", "payload is not a JSON object");
  }
  if (j.kind != JVal::kObj) Bad("Parse", "payload is not a JSON object");
  {
    const JVal& ver = Field(j, "version");
    if (ver.kind != JVal::kInt) Bad("Structure", "field version must be an integer");
    if (ver.i != 1) Bad("BadVersion", "unsupported version " + std::to_string(ver.i));
  }
  Automaton a;
  const int64_t S = IntField(j, "num_states");
  if (S < 1 || S > 1000000) Bad("Structure", "num_states out of range");
  a.num_states = static_cast<int32_t>(S);
  const int64_t initial = IntField(j, "initial_state");
  const int64_t accept = IntField(j, "accept_state");
  if (initial < 0 || initial >= S || accept < 0 || accept >= S) {
    Bad("Structure", "initial or accept state out of range");
  }
  a.initial_state = static_cast<int32_t>(initial);
  a.accept_state = static_cast<int32_t>(accept);
  a.grammar_text = StrField(j, "grammar_text");
  const std::string hash_hex = StrField(j, "grammar_hash");
  a.grammar_hash = GrammarHash(a.grammar_text);
  if (HashHex(a.grammar_hash) != hash_hex) Bad("Structure", "grammar hash does not match grammar text");

  a.shift_targets.assign(static_cast<size_t>(S) * 256, -1);
  const JVal& shifts = Field(j, "shifts");
  if (shifts.kind != JVal::kArr) Bad("Structure", "shifts must be an array");
  for (const JVal& row : shifts.arr) {
    if (row.kind != JVal::kArr || row.arr.size() != 3 || row.arr[0].kind != JVal::kInt ||
        row.arr[1].kind != JVal::kInt || row.arr[2].kind != JVal::kInt) {
      Bad("Structure", "shift rows must be [state, byte, target]");
    }
    const int64_t s = row.arr[0].i, b = row.arr[1].i, t = row.arr[2].i;
    if (s < 0 || s >= S || b < 0 || b > 255 || t < 0 || t >= S) Bad("Structure", "shift row out of range");
    a.shift_targets[static_cast<size_t>(s) * 256 + static_cast<size_t>(b)] = static_cast<int32_t>(t);
  }
  const JVal& edges = Field(j, "edges");
  if (edges.kind != JVal::kArr) Bad("Structure", "edges must be an array");
  for (const JVal& je : edges.arr) a.edges.push_back(EdgeOf(je, S, false));
  const JVal& comps = Field(j, "composites");
  if (comps.kind != JVal::kArr) Bad("Structure", "composites must be an array");
  for (const JVal& je : comps.arr) a.composite_edges.push_back(EdgeOf(je, S, true));
  const JVal& cycles = Field(j, "cycles");
  if (cycles.kind != JVal::kArr) Bad("Structure", "cycles must be an array");
  for (const JVal& jc : cycles.arr) {
    CycleRec c;
    const int64_t b = IntField(jc, "closing_byte");
    if (b < 0 || b > 255) Bad("Structure", "closing byte out of range");
    c.closing_byte = static_cast<int>(b);
    c.states = StateVec(jc, "states", S);
    if (c.states.empty()) Bad("Structure", "cycle without states");
    a.cycle_list.push_back(std::move(c));
  }
  const JVal& st = Field(j, "stats");
  a.stats.states = IntField(st, "states");
  a.stats.acceptance = IntField(st, "acceptance_edges");
  a.stats.reduction = IntField(st, "reduction_edges");
  a.stats.cycle_back = IntField(st, "cycle_back_edges");
  a.stats.merged = IntField(st, "merged_edges");
  a.stats.aggregated_groups = IntField(st, "aggregated_groups");
  a.stats.edges_before_aggregation = IntField(st, "edges_before_aggregation");
  // Arbitration order is never trusted from disk.
  try {
    FinalizeAndCheck(&a);
  } catch (const Error& e) {
    Bad("Structure", std::string("loaded machine is inconsistent: ") + e.what());
  }
  a.Validate();
  return a;
}

std::string EscapeToken(const std::string& s) {
  static const char* kHex = "0123456789abcdef";
  std::string out;
  for (char ch : s) {
    const unsigned char b = static_cast<unsigned char>(ch);
    if (ch == '\\') {
      out += "\\\\";
    } else if (b >= 0x20 && b <= 0x7e) {
      out.push_back(ch);
    } else {
      out += "\\x";
      out.push_back(kHex[b >> 4]);
      out.push_back(kHex[b & 0xf]);
    }
  }
  return out;
}

namespace {
std::string UnescapeToken(const std::string& s) {
  std::string out;
  for (size_t i = 0; i < s.size(); ++i) {
    if (s[i] != '\\') {
      out.push_back(s[i]);
      continue;
    }
    if (i + 1 >= s.size()) Bad("Parse", "dangling backslash in token");
    const char c = s[++i];
    if (c == '\\') {
      out.push_back('\\');
    } else if (c == 'x') {
      if (i + 2 >= s.size()) Bad("Parse", "truncated \\x escape in token");
      auto hex = [](char h) -> int {
        if (h >= '0' && h <= '9') return h - '0';
        if (h >= 'a' && h <= 'f') return h - 'a' + 10;
        if (h >= 'A' && h <= 'F') return h - 'A' + 10;
        Bad("Parse", "bad hex digit in \\x escape");
      };
      const int hi = hex(s[i + 1]);
      const int lo = hex(s[i + 2]);
      i += 2;
      out.push_back(static_cast<char>(hi * 16 + lo));
    } else {
      Bad("Parse", std::string("unknown escape \\") + c + " in token");
    }
  }
  return out;
}
}  // namespace

std::vector<std::string> LoadVocabularyJson(const uint8_t* data, size_t n) {
  const char* p = reinterpret_cast<const char*>(data);
  JVal j;
  try {
    j = ParseJson(p, p + n);
  } catch (const Error&) {
    Bad("Parse", "vocabulary must be a JSON array of strings");
  }
  if (j.kind != JVal::kArr) Bad("Parse", "vocabulary must be a JSON array of strings");
  std::vector<std::string> out;
  out.reserve(j.arr.size());
  for (const JVal& v : j.arr) {
    if (v.kind != JVal::kStr) Bad("Parse", "vocabulary entries must be strings");
    out.push_back(UnescapeToken(v.s));
  }
  return out;
}

}  // namespace pre3
