// compiler.cpp — host grammar compiler: BNF text -> canonical LR(1) ->
// DPDA with prefix-conditioned edges.
//
// Produces exactly the automaton the reference builds (same state numbering,
// same edges in the same arbitration order, same normalized grammar text and
// hash), so P3DPDA files from either side are byte-identical; the parity
// tests compare against the reference-built goldens and, in the build
// container, against the reference compiler itself.
//
// Stages and the reference behaviour each restates:
//   ParseText      ParseGrammar          grammar.cpp:113-185 (syntax, ids in
//                                        first-appearance order, errors)
//   Normalize      PrintGrammar + FNV-1a grammar.cpp:219-246, dpda_builder.cpp:469-476
//   FirstSets      ComputeFirstSets      grammar.cpp:270-320 (least fixpoint)
//   Collection     BuildCanonicalCollection lr1.cpp:138-214 (BFS numbering,
//                                        bytes ascending then nonterminals)
//   Tables         BuildTables           lr1.cpp:249-305 (conflict order)
//   ChainRunner    ChainSimulator        dpda_builder.cpp:116-255 (reduce
//                                        chains, downward branching, pumps)
//   FindCycles     DetectCycles          dpda_builder.cpp:340-364
//   Aggregate      AggregateEdges        optimizer.cpp:33-76
//   Order          EdgeOrderBefore / FinalizeEdgeOrder dpda_builder.cpp:327-338,450-467
//   CheckDeterminism ValidateDeterminism dpda_builder.cpp:409-448
//   MergeComposites  MergeEdges          optimizer.cpp:78-136 (composites are
//                                        sequence-runner only; GMASKDP1 keeps them)
//
// Data structures are this file's own: 257-bit terminal sets in five words,
// item sets as sorted (core, lookahead) arrays hashed by content, the action
// table as one packed int per (state, terminal).
#include <algorithm>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <tuple>
#include <unordered_map>
#include <utility>
#include <vector>

#include "gm_internal.hpp"

namespace pre3 {
namespace {

constexpr int kEnd = 256;       // $ terminal
constexpr int kNt0 = 257;       // first nonterminal id
constexpr int64_t kStateCeiling = 1000000;
constexpr int64_t kEdgeBudgetFactor = 100;

[[noreturn]] void GrammarFail(const std::string& m) { throw Error(GM_ERR_GRAMMAR, m); }
[[noreturn]] void BuildFail(const std::string& m) { throw Error(GM_ERR_BUILD, m); }

// ---------------------------------------------------------------- sets
// Terminal set over bytes 0..255 plus $ (bit 256).
struct TSet {
  uint64_t w[5] = {0, 0, 0, 0, 0};
  void Add(int t) { w[t >> 6] |= 1ull << (t & 63); }
  bool Has(int t) const { return (w[t >> 6] >> (t & 63)) & 1ull; }
  bool None() const { return (w[0] | w[1] | w[2] | w[3] | w[4]) == 0; }
  bool Merge(const TSet& o) {
    bool grew = false;
    for (int i = 0; i < 5; ++i) {
      const uint64_t n = w[i] | o.w[i];
      grew |= n != w[i];
      w[i] = n;
    }
    return grew;
  }
  int Count() const {
    int n = 0;
    for (uint64_t x : w) n += __builtin_popcountll(x);
    return n;
  }
  bool operator==(const TSet& o) const { return std::memcmp(w, o.w, sizeof(w)) == 0; }
  template <typename F>
  void Each(F&& f) const {  // ascending; $ last
    for (int i = 0; i < 5; ++i) {
      for (uint64_t x = w[i]; x; x &= x - 1) f(i * 64 + __builtin_ctzll(x));
    }
  }
};

std::string ByteLabel(int b) {
  if (b == kEnd) return "$";
  std::string s = "'";
  const unsigned char c = static_cast<unsigned char>(b);
  if (c == '"' || c == '\\') {
    s += '\\';
    s += static_cast<char>(c);
  } else if (c >= 0x20 && c < 0x7f) {
    s += static_cast<char>(c);
  } else {
    char buf[8];
    std::snprintf(buf, sizeof(buf), "\\x%02x", c);
    s += buf;
  }
  return s + "'";
}

std::string StackText(const std::vector<int32_t>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}

// ---------------------------------------------------------------- grammar
struct Cfg {
  std::vector<int32_t> lhs;                 // per production
  std::vector<std::vector<int32_t>> rhs;    // per production; 0..255 bytes, >= 257 nonterminals
  std::vector<std::string> names;           // per nonterminal
  std::vector<std::vector<int32_t>> prods;  // per nonterminal, declaration order
  int32_t start = kNt0;
  int32_t aug = -1;  // augmented production id
  int NumNt() const { return static_cast<int>(names.size()); }
  int NumProd() const { return static_cast<int>(lhs.size()); }
};

struct LineCursor {
  const std::string& s;
  int line;
  size_t i = 0;
  bool Done() const { return i >= s.size(); }
  void Blank() {
    while (!Done() && (s[i] == ' ' || s[i] == '\t')) ++i;
  }
  [[noreturn]] void Fail(const std::string& m) const {
    GrammarFail("MalformedGrammar: line " + std::to_string(line) + ", column " + std::to_string(i + 1) + ": " + m);
  }
};

bool IdHead(char c) { return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_'; }
bool IdTail(char c) { return IdHead(c) || (c >= '0' && c <= '9'); }

int Hex(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

std::string Identifier(LineCursor& c) {
  if (c.Done() || !IdHead(c.s[c.i])) c.Fail("expected identifier");
  const size_t b = c.i;
  while (!c.Done() && IdTail(c.s[c.i])) ++c.i;
  return c.s.substr(b, c.i - b);
}

// Quoted literal at c.i (opening quote) -> its bytes.
std::string Literal(LineCursor& c) {
  ++c.i;
  std::string out;
  for (;;) {
    if (c.Done()) c.Fail("unterminated terminal literal");
    const char ch = c.s[c.i];
    if (ch == '"') {
      ++c.i;
      break;
    }
    if (ch != '\\') {
      out += ch;
      ++c.i;
      continue;
    }
    ++c.i;
    if (c.Done()) c.Fail("dangling escape");
    const char e = c.s[c.i];
    if (e == '"' || e == '\\') {
      out += e;
      ++c.i;
    } else if (e == 'x') {
      if (c.i + 2 >= c.s.size()) c.Fail("truncated \\xNN escape");
      const int hi = Hex(c.s[c.i + 1]), lo = Hex(c.s[c.i + 2]);
      if (hi < 0 || lo < 0) c.Fail("bad hex digits in \\xNN escape");
      out += static_cast<char>(hi * 16 + lo);
      c.i += 3;
    } else {
      c.Fail(std::string("unknown escape \\") + e);
    }
  }
  if (out.empty()) c.Fail("empty terminal literal");
  return out;
}

// Cuts a '#' comment that is not inside a literal.
std::string Uncomment(const std::string& line) {
  bool in_lit = false;
  for (size_t i = 0; i < line.size(); ++i) {
    const char ch = line[i];
    if (in_lit) {
      if (ch == '\\') ++i;
      else if (ch == '"') in_lit = false;
    } else if (ch == '"') {
      in_lit = true;
    } else if (ch == '#') {
      return line.substr(0, i);
    }
  }
  return line;
}

Cfg ParseText(const std::string& text) {
  Cfg g;
  std::map<std::string, int32_t> id_of;
  auto nt = [&](const std::string& name) {
    auto it = id_of.find(name);
    if (it != id_of.end()) return it->second;
    const int32_t id = kNt0 + g.NumNt();
    g.names.push_back(name);
    g.prods.emplace_back();
    id_of.emplace(name, id);
    return id;
  };
  // std::getline semantics: '\n' separated, a trailing newline adds no line.
  size_t pos = 0;
  int line_no = 0;
  bool first = true;
  while (pos < text.size()) {
    size_t nl = text.find('\n', pos);
    if (nl == std::string::npos) nl = text.size();
    const std::string line = Uncomment(text.substr(pos, nl - pos));
    pos = nl + 1;
    ++line_no;
    LineCursor c{line, line_no};
    c.Blank();
    if (c.Done()) continue;
    const std::string head = Identifier(c);
    c.Blank();
    if (c.i + 1 >= line.size() || line[c.i] != '-' || line[c.i + 1] != '>') c.Fail("expected '->' after rule name");
    c.i += 2;
    const int32_t lhs = nt(head);
    if (first) {
      g.start = lhs;
      first = false;
    }
    std::vector<int32_t> alt;
    auto close_alt = [&]() {
      g.prods[lhs - kNt0].push_back(g.NumProd());
      g.lhs.push_back(lhs);
      g.rhs.push_back(alt);
      alt.clear();
    };
    for (;;) {
      c.Blank();
      if (c.Done()) break;
      const char ch = c.s[c.i];
      if (ch == '|') {
        close_alt();
        ++c.i;
      } else if (ch == '"') {
        for (char b : Literal(c)) alt.push_back(static_cast<unsigned char>(b));
      } else if (IdHead(ch)) {
        alt.push_back(nt(Identifier(c)));
      } else {
        c.Fail(std::string("unexpected character '") + ch + "'");
      }
    }
    close_alt();
  }
  if (g.lhs.empty()) GrammarFail("EmptyGrammar: no rules found");
  for (const auto& r : g.rhs) {
    for (int32_t s : r) {
      if (s >= kNt0 && g.prods[s - kNt0].empty()) {
        GrammarFail("UndefinedSymbol: '" + g.names[s - kNt0] + "' is used but has no rule");
      }
    }
  }
  return g;
}

void Augment(Cfg* g) {
  const int32_t id = kNt0 + g->NumNt();
  g->names.push_back(g->names[g->start - kNt0] + "'");
  g->aug = g->NumProd();
  g->prods.push_back({g->aug});
  g->lhs.push_back(id);
  g->rhs.push_back({g->start});
}

std::string Escape(const std::string& bytes) {
  std::string out;
  for (char ch : bytes) {
    const unsigned char u = static_cast<unsigned char>(ch);
    if (ch == '"' || ch == '\\') {
      out += '\\';
      out += ch;
    } else if (u >= 0x20 && u < 0x7f) {
      out += ch;
    } else {
      char buf[8];
      std::snprintf(buf, sizeof(buf), "\\x%02x", u);
      out += buf;
    }
  }
  return out;
}

// One production per line, runs of bytes re-quoted (the reparseable text the
// automaton carries and hashes).
std::string Normalize(const Cfg& g) {
  std::string out;
  for (int p = 0; p < g.NumProd(); ++p) {
    if (p == g.aug) continue;
    out += g.names[g.lhs[p] - kNt0] + " ->";
    std::string run;
    for (int32_t s : g.rhs[p]) {
      if (s < 256) {
        run += static_cast<char>(s);
        continue;
      }
      if (!run.empty()) out += " \"" + Escape(run) + "\"";
      run.clear();
      out += " " + g.names[s - kNt0];
    }
    if (!run.empty()) out += " \"" + Escape(run) + "\"";
    out += "\n";
  }
  return out;
}

uint64_t Fnv1a(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (char ch : s) h = (h ^ static_cast<unsigned char>(ch)) * 0x100000001b3ull;
  return h;
}

// ---------------------------------------------------------------- FIRST
struct First {
  std::vector<TSet> set;     // per nonterminal (bytes; never $)
  std::vector<char> eps;     // per nonterminal: nullable
  // FIRST(seq . tail) for a non-empty-lookahead tail.
  TSet OfSeq(const Cfg&, const int32_t* seq, size_t n, const TSet& tail) const {
    TSet out;
    for (size_t i = 0; i < n; ++i) {
      const int32_t s = seq[i];
      if (s < 256) {
        out.Add(s);
        return out;
      }
      out.Merge(set[s - kNt0]);
      if (!eps[s - kNt0]) return out;
    }
    out.Merge(tail);
    return out;
  }
};

First FirstSets(const Cfg& g) {
  First f;
  f.set.assign(g.NumNt(), TSet{});
  f.eps.assign(g.NumNt(), 0);
  for (bool again = true; again;) {
    again = false;
    for (int p = 0; p < g.NumProd(); ++p) {
      const int a = g.lhs[p] - kNt0;
      bool all_eps = true;
      for (int32_t s : g.rhs[p]) {
        if (s < 256) {
          TSet t;
          t.Add(s);
          again |= f.set[a].Merge(t);
          all_eps = false;
          break;
        }
        again |= f.set[a].Merge(f.set[s - kNt0]);
        if (!f.eps[s - kNt0]) {
          all_eps = false;
          break;
        }
      }
      if (all_eps && !f.eps[a]) {
        f.eps[a] = 1;
        again = true;
      }
    }
  }
  return f;
}

// ---------------------------------------------------------------- LR(1)
// Item set: cores (production, dot) sorted ascending, one lookahead set each.
struct Items {
  std::vector<std::pair<int32_t, int32_t>> core;
  std::vector<TSet> la;
  bool operator==(const Items& o) const { return core == o.core && la == o.la; }
  uint64_t Hash() const {
    uint64_t h = 0x243f6a8885a308d3ull;
    auto mix = [&h](uint64_t v) { h = (h ^ v) * 0x100000001b3ull + (h >> 29); };
    for (size_t i = 0; i < core.size(); ++i) {
      mix((static_cast<uint64_t>(core[i].first) << 32) | static_cast<uint32_t>(core[i].second));
      for (uint64_t x : la[i].w) mix(x);
    }
    return h;
  }
};

// Least closed superset: [B -> .gamma, FIRST(beta a)] for every
// [A -> alpha . B beta, a] (lr1.cpp:86-111).
Items Close(const Cfg& g, const First& f, const std::vector<std::pair<int32_t, int32_t>>& kcore,
            const std::vector<TSet>& kla) {
  std::unordered_map<int64_t, int> at;
  std::vector<std::pair<int32_t, int32_t>> core = kcore;
  std::vector<TSet> la = kla;
  std::vector<int> queue;
  std::vector<char> queued;
  for (size_t i = 0; i < core.size(); ++i) {
    at.emplace((static_cast<int64_t>(core[i].first) << 32) | core[i].second, static_cast<int>(i));
    queue.push_back(static_cast<int>(i));
    queued.push_back(1);
  }
  for (size_t qi = 0; qi < queue.size(); ++qi) {
    const int i = queue[qi];
    queued[i] = 0;
    const auto [p, dot] = core[i];
    const auto& r = g.rhs[p];
    if (dot >= static_cast<int>(r.size()) || r[dot] < kNt0) continue;
    const TSet follow = f.OfSeq(g, r.data() + dot + 1, r.size() - dot - 1, la[i]);
    if (follow.None()) continue;  // an item needs a lookahead (lr1.cpp:15, ItemSet::Add)
    for (int32_t q : g.prods[r[dot] - kNt0]) {
      const int64_t key = static_cast<int64_t>(q) << 32;
      auto it = at.find(key);
      int j;
      bool grew;
      if (it == at.end()) {
        j = static_cast<int>(core.size());
        at.emplace(key, j);
        core.emplace_back(q, 0);
        la.push_back(follow);
        queued.push_back(0);
        grew = true;
      } else {
        j = it->second;
        grew = la[j].Merge(follow);
      }
      if (grew && !queued[j]) {
        queued[j] = 1;
        queue.push_back(j);
      }
    }
  }
  std::vector<int> order(core.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return core[a] < core[b]; });
  Items out;
  for (int i : order) {
    out.core.push_back(core[i]);
    out.la.push_back(la[i]);
  }
  return out;
}

struct Lr1 {
  std::vector<Items> states;
  std::vector<std::vector<std::pair<int32_t, int32_t>>> trans;  // (symbol, target), symbol order
  std::vector<std::vector<std::pair<int32_t, int32_t>>> reduce;  // (production, terminal) sorted
  std::vector<std::vector<int32_t>> preds;                       // ascending, unique
  std::vector<int32_t> access;                                   // accessing symbol, -1 for 0
  int32_t accept = -1;
  int32_t Goto(int32_t s, int32_t x) const {
    for (const auto& [sym, t] : trans[s]) {
      if (sym == x) return t;
    }
    return -1;
  }
  int32_t S() const { return static_cast<int32_t>(states.size()); }
};

Lr1 Collection(const Cfg& g, const First& f) {
  Lr1 m;
  std::unordered_map<uint64_t, std::vector<int32_t>> by_hash;
  auto intern = [&](Items&& it, int32_t sym, bool* fresh) {
    const uint64_t h = it.Hash();
    auto& bucket = by_hash[h];
    for (int32_t id : bucket) {
      if (m.states[id] == it) {
        *fresh = false;
        return id;
      }
    }
    const int32_t id = m.S();
    if (id >= kStateCeiling) {
      BuildFail("StateExplosion: canonical collection exceeded ceiling of " + std::to_string(kStateCeiling) +
                " states");
    }
    m.states.push_back(std::move(it));
    m.access.push_back(sym);
    bucket.push_back(id);
    *fresh = true;
    return id;
  };
  {
    TSet end;
    end.Add(kEnd);
    bool fresh;
    intern(Close(g, f, {{g.aug, 0}}, {end}), -1, &fresh);
  }
  for (int32_t s = 0; s < m.S(); ++s) {  // FIFO over ids = BFS order
    const Items cur = m.states[s];
    // Symbols after a dot: bytes ascending, then nonterminals by id.
    std::vector<char> seen(256 + 1 + g.NumNt(), 0);
    for (size_t i = 0; i < cur.core.size(); ++i) {
      const auto& r = g.rhs[cur.core[i].first];
      if (cur.core[i].second < static_cast<int>(r.size())) seen[r[cur.core[i].second]] = 1;
    }
    std::vector<std::pair<int32_t, int32_t>> out;
    for (int32_t x = 0; x < static_cast<int32_t>(seen.size()); ++x) {
      if (!seen[x]) continue;
      std::vector<std::pair<int32_t, int32_t>> kc;
      std::vector<TSet> kl;
      for (size_t i = 0; i < cur.core.size(); ++i) {
        const auto [p, dot] = cur.core[i];
        if (dot < static_cast<int>(g.rhs[p].size()) && g.rhs[p][dot] == x) {
          kc.emplace_back(p, dot + 1);  // stays sorted: cores are sorted by (p, dot)
          kl.push_back(cur.la[i]);
        }
      }
      bool fresh;
      const int32_t t = intern(Close(g, f, kc, kl), x, &fresh);
      out.emplace_back(x, t);
    }
    m.trans.push_back(std::move(out));
  }
  const int32_t S = m.S();
  m.reduce.resize(S);
  m.preds.resize(S);
  for (int32_t s = 0; s < S; ++s) {
    const Items& it = m.states[s];
    for (size_t i = 0; i < it.core.size(); ++i) {
      const auto [p, dot] = it.core[i];
      if (dot != static_cast<int>(g.rhs[p].size())) continue;
      if (p == g.aug) {
        m.accept = s;
        continue;
      }
      it.la[i].Each([&](int t) { m.reduce[s].emplace_back(p, t); });
    }
    std::sort(m.reduce[s].begin(), m.reduce[s].end());
    for (const auto& tr : m.trans[s]) m.preds[tr.second].push_back(s);
  }
  for (auto& v : m.preds) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  return m;
}

// ACTION cell: 0 error; kShift|target; kReduce|production; kAcceptCell.
constexpr int32_t kShift = 1 << 28, kReduce = 2 << 28, kAcceptCell = 3 << 28, kKindMask = 3 << 28;

struct Tables {
  std::vector<int32_t> act;  // S*257
  int32_t At(int32_t s, int t) const { return act[static_cast<size_t>(s) * 257 + t]; }
};

std::string CellText(const Cfg& g, int32_t c) {
  const int32_t v = c & ~kKindMask;
  switch (c & kKindMask) {
    case kShift: return "shift to state " + std::to_string(v);
    case kReduce: return "reduce by " + g.names[g.lhs[v] - kNt0] + " (production " + std::to_string(v) + ")";
    case kAcceptCell: return "accept";
  }
  return "error";
}

Tables BuildTables(const Cfg& g, const Lr1& m) {
  Tables t;
  t.act.assign(static_cast<size_t>(m.S()) * 257, 0);
  auto put = [&](int32_t s, int term, int32_t cell) {
    int32_t& c = t.act[static_cast<size_t>(s) * 257 + term];
    if (c != 0 && c != cell) {
      BuildFail("NotLR1Conflict: state " + std::to_string(s) + " on " + ByteLabel(term) + ": " + CellText(g, c) +
                " vs " + CellText(g, cell));
    }
    c = cell;
  };
  for (int32_t s = 0; s < m.S(); ++s) {
    for (const auto& [x, tgt] : m.trans[s]) {
      if (x < 256) put(s, x, kShift | tgt);
    }
    for (const auto& [p, term] : m.reduce[s]) put(s, term, kReduce | p);
    if (s == m.accept) put(s, kEnd, kAcceptCell);
  }
  return t;
}

// ---------------------------------------------------------------- edges
struct BEdge {
  int32_t src = -1;
  TSet acc;                   // bytes + $
  TSet acc2;                  // composites: second terminal
  std::vector<int32_t> pop;   // top first
  std::vector<int32_t> push;  // bottom first
  int32_t target = -1;
  uint8_t origin = 0;  // 0 acceptance, 1 reduction, 2 cycle back, 3 merged (dpda.hpp:35)
  bool dyn = false;
};

int Rank(uint8_t origin) {  // arbitration rank (dpda_builder.cpp:20-28)
  static const int r[4] = {2, 1, 0, 3};
  return r[origin & 3];
}

// EdgeOrderBefore (dpda_builder.cpp:327-338): source; longer condition; rank;
// condition lexicographic; without-$ first; accepted bytes by their hex image
// (nibble 0 of word 0 first).
bool Before(const BEdge& a, const BEdge& b) {
  if (a.src != b.src) return a.src < b.src;
  if (a.pop.size() != b.pop.size()) return a.pop.size() > b.pop.size();
  const int ra = Rank(a.origin), rb = Rank(b.origin);
  if (ra != rb) return ra < rb;
  if (a.pop != b.pop) return a.pop < b.pop;
  const bool da = a.acc.Has(kEnd), db = b.acc.Has(kEnd);
  if (da != db) return db;
  for (int n = 0; n < 64; ++n) {
    const unsigned x = (a.acc.w[n >> 4] >> ((n & 15) * 4)) & 15u;
    const unsigned y = (b.acc.w[n >> 4] >> ((n & 15) * 4)) & 15u;
    if (x != y) return x < y;
  }
  return false;
}

// Pump-free reduce-chain simulation (one instance per run).
struct ChainRunner {
  const Cfg& g;
  const Lr1& m;
  const Tables& tab;
  const std::vector<std::vector<int32_t>>& cycles;  // bottom first, entry first
  std::vector<BEdge>* edges = nullptr;              // emit target (null: pump search)
  std::vector<std::vector<int32_t>>* pumps = nullptr;
  int64_t edge_budget = 0;
  size_t depth_budget = 0;

  struct Hist {
    int32_t state, bottom;
    std::vector<int32_t> stack;
    size_t depth;
  };
  struct Branch {
    std::vector<int32_t> matched;  // original-stack suffix, top first
    std::vector<int32_t> cur;      // present stack above the unknown part, top first
    int32_t state;
    std::vector<Hist> hist;
  };

  // The matched suffix (bottom first) must not contain a rewritten circuit
  // followed by its own entry state (dpda_builder.cpp:82-104).
  bool Allowed(const std::vector<int32_t>& matched) const {
    const size_t L = matched.size();
    for (const auto& c : cycles) {
      const size_t n = c.size();
      if (L < n + 1) continue;
      for (size_t st = 0; st + n + 1 <= L; ++st) {
        // bottom-first index k corresponds to matched[L-1-k]
        bool hit = true;
        for (size_t i = 0; i < n && hit; ++i) hit = matched[L - 1 - (st + i)] == c[i];
        if (hit && matched[L - 1 - (st + n)] == c[0]) return false;
      }
    }
    return true;
  }

  void Run() {
    edge_budget = kEdgeBudgetFactor * static_cast<int64_t>(m.S()) * 257;
    depth_budget = static_cast<size_t>(m.S()) * 4 + 16;
    for (int32_t s = 0; s < m.S(); ++s) {
      for (const auto& pr : m.reduce[s]) Seed(s, pr.second);
    }
  }

  void Seed(int32_t seed, int la) {
    std::vector<Branch> work;  // LIFO (dpda_builder.cpp:133-140)
    work.push_back(Branch{{seed}, {seed}, seed, {}});
    while (!work.empty()) {
      Branch br = std::move(work.back());
      work.pop_back();
      Advance(seed, la, std::move(br), &work);
    }
  }

  void Emit(int32_t seed, int la, const Branch& br, int32_t shift_to) {
    if (edges == nullptr) return;
    if (static_cast<int64_t>(edges->size()) >= edge_budget) {
      BuildFail("StateExplosion: edge budget exceeded at " + std::to_string(edges->size()) + " edges");
    }
    BEdge e;
    e.src = seed;
    e.origin = 1;
    e.acc.Add(la);
    e.pop = br.matched;
    e.push.assign(br.cur.rbegin(), br.cur.rend());
    if (shift_to >= 0) {
      e.push.push_back(shift_to);
      e.target = shift_to;
    } else {
      e.target = m.accept;
    }
    edges->push_back(std::move(e));
  }

  void Advance(int32_t seed, int la, Branch br, std::vector<Branch>* work) {
    const int32_t cell = tab.At(br.state, la);
    switch (cell & kKindMask) {
      case 0: return;  // the lookahead never follows this context
      case kShift: Emit(seed, la, br, cell & ~kKindMask); return;
      case kAcceptCell: Emit(seed, la, br, -1); return;
      default: break;
    }
    const int32_t p = cell & ~kKindMask;
    const size_t r = g.rhs[p].size();
    if (br.cur.size() < r + 1) {
      // The state under the handle is unknown: branch over predecessors.
      if (br.matched.size() >= depth_budget) {
        BuildFail("DivergentReduction: reduce chain at state " + std::to_string(seed) + " exceeded depth budget " +
                  std::to_string(depth_budget));
      }
      for (int32_t pr : m.preds[br.matched.back()]) {
        Branch nb = br;
        nb.matched.push_back(pr);
        nb.cur.push_back(pr);
        if (Allowed(nb.matched)) work->push_back(std::move(nb));
      }
      return;
    }
    for (const Hist& h : br.hist) {
      if (h.state == br.state && h.bottom == br.matched.back() && h.depth < br.matched.size() && h.stack == br.cur) {
        std::vector<int32_t> circuit(br.matched.rbegin(), br.matched.rend() - static_cast<int64_t>(h.depth));
        if (pumps != nullptr) {
          pumps->push_back(std::move(circuit));
          return;
        }
        BuildFail("DivergentReduction: unrewritten pump at state " + std::to_string(seed) + " via circuit " +
                  StackText(circuit));
      }
    }
    br.hist.push_back(Hist{br.state, br.matched.back(), br.cur, br.matched.size()});
    br.cur.erase(br.cur.begin(), br.cur.begin() + static_cast<int64_t>(r));
    const int32_t nxt = m.Goto(br.cur.front(), g.lhs[p]);
    if (nxt < 0) return;
    br.cur.insert(br.cur.begin(), nxt);
    br.state = nxt;
    if (br.cur.size() > depth_budget) {
      BuildFail("DivergentReduction: simulated stack at state " + std::to_string(seed) + " exceeded depth budget " +
                std::to_string(depth_budget));
    }
    work->push_back(std::move(br));
  }
};

// Primitive period, then rotation to the smallest state (dpda_builder.cpp:59-77).
std::vector<int32_t> Canonical(std::vector<int32_t> c) {
  for (size_t per = 1; per < c.size(); ++per) {
    if (c.size() % per) continue;
    bool rep = true;
    for (size_t i = per; i < c.size() && rep; ++i) rep = c[i] == c[i - per];
    if (rep) {
      c.resize(per);
      break;
    }
  }
  const auto lo = std::min_element(c.begin(), c.end());
  std::rotate(c.begin(), lo, c.end());
  return c;
}

struct Circuit {
  std::vector<int32_t> states;  // bottom first
  int closing = 0;
};

Circuit MakeCircuit(const Lr1& m, std::vector<int32_t> states) {
  for (int32_t s : states) {
    if (m.access[s] < 0 || m.access[s] >= 256) {
      BuildFail("DivergentReduction: pumping circuit " + StackText(states) + " passes through state " +
                std::to_string(s) + " reached by a nonterminal; no stack rewrite preserves the language");
    }
  }
  Circuit c;
  c.closing = -1;
  for (const auto& [x, t] : m.trans[states.back()]) {
    if (x < 256 && t == states.front()) {
      c.closing = x;
      break;
    }
  }
  if (c.closing < 0) BuildFail("DivergentReduction: circuit " + StackText(states) + " has no closing byte transition");
  c.states = std::move(states);
  return c;
}

std::vector<Circuit> FindCycles(const Cfg& g, const Lr1& m, const Tables& tab) {
  std::vector<Circuit> out;
  std::vector<std::vector<int32_t>> known;
  for (;;) {
    std::vector<std::vector<int32_t>> pumps;
    ChainRunner run{g, m, tab, known};
    run.pumps = &pumps;
    run.Run();
    bool added = false;
    for (auto& p : pumps) {
      std::vector<int32_t> c = Canonical(std::move(p));
      if (std::find(known.begin(), known.end(), c) != known.end()) continue;
      out.push_back(MakeCircuit(m, c));
      known.push_back(std::move(c));
      added = true;
    }
    if (!added) break;
    for (size_t i = 0; i < out.size(); ++i) {
      for (size_t j = i + 1; j < out.size(); ++j) {
        for (int32_t s : out[i].states) {
          if (std::find(out[j].states.begin(), out[j].states.end(), s) != out[j].states.end()) {
            throw Error(GM_ERR_BUILD, "OverlappingCycles: circuits " + StackText(out[i].states) + " and " +
                                          StackText(out[j].states) + " share state " + std::to_string(s));
          }
        }
      }
    }
  }
  return out;
}

// Groups single-byte shift-tailed edges by (source, origin, condition, push
// prefix) into dynamic-target edges (optimizer.cpp:17-76).
int64_t Aggregate(const std::vector<int32_t>& shift, std::vector<BEdge>* edges) {
  using Key = std::tuple<int32_t, int, std::vector<int32_t>, std::vector<int32_t>>;
  std::map<Key, std::vector<size_t>> groups;
  std::vector<int> byte(edges->size(), -1);
  for (size_t i = 0; i < edges->size(); ++i) {
    const BEdge& e = (*edges)[i];
    if (e.dyn || e.acc.Has(kEnd) || e.origin == 3 || e.acc.Count() != 1) continue;
    if (e.push.size() < 2 || e.push.back() != e.target) continue;
    int b = -1;
    e.acc.Each([&](int t) { b = t; });
    if (shift[static_cast<size_t>(e.push[e.push.size() - 2]) * 256 + b] != e.target) continue;
    byte[i] = b;
    groups[Key{e.src, e.origin, e.pop, std::vector<int32_t>(e.push.begin(), e.push.end() - 1)}].push_back(i);
  }
  std::vector<char> gone(edges->size(), 0);
  std::vector<BEdge> made;
  for (const auto& [key, members] : groups) {
    if (members.size() < 2) continue;
    BEdge d;
    const BEdge& f = (*edges)[members.front()];
    d.src = f.src;
    d.pop = f.pop;
    d.push.assign(f.push.begin(), f.push.end() - 1);
    d.origin = f.origin;
    d.dyn = true;
    d.target = -1;
    for (size_t i : members) {
      d.acc.Add(byte[i]);
      gone[i] = 1;
    }
    made.push_back(std::move(d));
  }
  if (made.empty()) return 0;
  const int64_t rewritten = static_cast<int64_t>(made.size());
  std::vector<BEdge> kept;
  for (size_t i = 0; i < edges->size(); ++i) {
    if (!gone[i]) kept.push_back(std::move((*edges)[i]));
  }
  for (BEdge& d : made) kept.push_back(std::move(d));
  edges->swap(kept);
  return rewritten;
}

void CheckDeterminism(const std::vector<int32_t>& shift, int32_t accept, const std::vector<BEdge>& e,
                      const std::vector<int32_t>& begin) {
  auto fail = [](const std::string& m) { BuildFail("NondeterministicEdges: " + m); };
  for (size_t s = 0; s + 1 < begin.size(); ++s) {
    for (int32_t i = begin[s]; i < begin[s + 1]; ++i) {
      const BEdge& x = e[i];
      if (x.pop.empty() || x.pop[0] != static_cast<int32_t>(s)) {
        fail("edge at state " + std::to_string(s) + " conditions on " + StackText(x.pop));
      }
      if (x.dyn) {
        bool bad = x.acc.Has(kEnd);
        x.acc.Each([&](int t) {
          if (t < 256 && (x.push.empty() || shift[static_cast<size_t>(x.push.back()) * 256 + t] < 0)) bad = true;
        });
        if (bad) fail("dynamic edge at state " + std::to_string(s) + " cannot resolve");
      } else if (x.push.empty() && x.target != accept) {
        fail("edge at state " + std::to_string(s) + " pushes nothing");
      }
    }
    for (int32_t i = begin[s]; i < begin[s + 1]; ++i) {
      for (int32_t j = i + 1; j < begin[s + 1]; ++j) {
        const BEdge& a = e[i];
        const BEdge& b = e[j];
        if (a.pop != b.pop || Rank(a.origin) != Rank(b.origin)) continue;
        bool common = false;
        for (int w = 0; w < 5; ++w) common |= (a.acc.w[w] & b.acc.w[w]) != 0;
        if (common) {
          fail("state " + std::to_string(s) + ": two rank-equal edges on " + StackText(a.pop) +
               " accept a common terminal");
        }
      }
    }
  }
}

// MergeEdges (optimizer.cpp:78-136): an edge whose target has exactly one
// outgoing edge composes with it into one two-terminal edge; composites are
// sequence-runner only (never read by Step / ComputeMask) and are kept for the
// GMASKDP1 format.  `e` is in finalized order; output in generation order.
std::vector<BEdge> MergeComposites(const std::vector<BEdge>& e, int32_t S, int32_t accept) {
  std::vector<int32_t> outdeg(S, 0), only(S, -1);
  std::vector<TSet> collapse(S);
  for (size_t i = 0; i < e.size(); ++i) {
    outdeg[e[i].src]++;
    only[e[i].src] = static_cast<int32_t>(i);
    if (e[i].origin == 2) collapse[e[i].src].Merge(e[i].acc);
  }
  std::vector<BEdge> out;
  for (const BEdge& a : e) {
    if (a.dyn || a.acc.Has(kEnd) || a.target < 0 || a.target == accept || outdeg[a.target] != 1) continue;
    bool clash = false;
    for (int w = 0; w < 4; ++w) clash |= (a.acc.w[w] & collapse[a.src].w[w]) != 0;
    if (clash) continue;
    const BEdge& b = e[only[a.target]];
    if (b.dyn) continue;
    const size_t k = std::min(b.pop.size(), a.push.size());
    bool ok = true;
    for (size_t i = 0; i < k && ok; ++i) ok = b.pop[i] == a.push[a.push.size() - 1 - i];
    if (!ok) continue;
    BEdge c;
    c.src = a.src;
    c.origin = 3;
    c.acc = a.acc;
    c.acc2 = b.acc;
    c.pop = a.pop;
    c.pop.insert(c.pop.end(), b.pop.begin() + static_cast<int64_t>(k), b.pop.end());
    c.push.assign(a.push.begin(), a.push.end() - static_cast<int64_t>(k));
    c.push.insert(c.push.end(), b.push.begin(), b.push.end());
    c.target = b.target;
    out.push_back(std::move(c));
  }
  return out;
}

Edge ToEdge(const BEdge& e) {
  Edge o;
  o.source = e.src;
  std::memcpy(o.accepted, e.acc.w, sizeof(o.accepted));
  o.dollar = e.acc.Has(kEnd);
  o.origin = e.origin;
  o.dynamic = e.dyn;
  o.target = e.target;
  o.match_pop = e.pop;
  o.push = e.push;
  std::memcpy(o.second, e.acc2.w, sizeof(o.second));
  o.dollar_second = e.acc2.Has(kEnd);
  return o;
}

BEdge FromEdge(const Edge& o) {
  BEdge e;
  e.src = o.source;
  std::memcpy(e.acc.w, o.accepted, sizeof(o.accepted));
  if (o.dollar) e.acc.Add(kEnd);
  std::memcpy(e.acc2.w, o.second, sizeof(o.second));
  if (o.dollar_second) e.acc2.Add(kEnd);
  e.origin = o.origin;
  e.dyn = o.dynamic;
  e.target = o.target;
  e.pop = o.match_pop;
  e.push = o.push;
  return e;
}

std::vector<int32_t> Ranges(const std::vector<BEdge>& edges, int32_t S) {
  std::vector<int32_t> begin(static_cast<size_t>(S) + 1, 0);
  for (const BEdge& e : edges) begin[e.src + 1]++;
  for (int32_t s = 0; s < S; ++s) begin[s + 1] += begin[s];
  return begin;
}

}  // namespace

Automaton CompileGrammar(const std::string& text, bool aggregate, bool merge) {
  Cfg g = ParseText(text);
  Augment(&g);
  const First f = FirstSets(g);
  const Lr1 m = Collection(g, f);
  const Tables tab = BuildTables(g, m);
  const int32_t S = m.S();

  Automaton a;
  a.num_states = S;
  a.initial_state = 0;
  a.accept_state = m.accept;
  a.grammar_text = Normalize(g);
  a.grammar_hash = Fnv1a(a.grammar_text);
  a.shift_targets.assign(static_cast<size_t>(S) * 256, -1);
  for (int32_t s = 0; s < S; ++s) {
    for (const auto& [x, t] : m.trans[s]) {
      if (x < 256) a.shift_targets[static_cast<size_t>(s) * 256 + x] = t;
    }
  }

  const std::vector<Circuit> cycles = FindCycles(g, m, tab);
  std::vector<BEdge> edges;
  for (int32_t s = 0; s < S; ++s) {  // acceptance: one plain shift per (state, byte)
    for (const auto& [x, t] : m.trans[s]) {
      if (x >= 256) continue;
      BEdge e;
      e.src = s;
      e.acc.Add(x);
      e.pop = {s};
      e.push = {s, t};
      e.target = t;
      e.origin = 0;
      edges.push_back(std::move(e));
    }
  }
  std::vector<std::vector<int32_t>> circuits;
  for (const Circuit& c : cycles) {  // cycle back: collapse the full circuit
    BEdge e;
    e.src = c.states.back();
    e.acc.Add(c.closing);
    e.pop.assign(c.states.rbegin(), c.states.rend());
    e.push = {c.states.front()};
    e.target = c.states.front();
    e.origin = 2;
    edges.push_back(std::move(e));
    circuits.push_back(c.states);
  }
  {
    ChainRunner run{g, m, tab, circuits};
    run.edges = &edges;
    run.Run();
  }
  a.stats.states = S;
  for (const BEdge& e : edges) {
    a.stats.acceptance += e.origin == 0;
    a.stats.reduction += e.origin == 1;
    a.stats.cycle_back += e.origin == 2;
  }
  a.stats.edges_before_aggregation = static_cast<int64_t>(edges.size());
  if (aggregate) a.stats.aggregated_groups = Aggregate(a.shift_targets, &edges);
  std::sort(edges.begin(), edges.end(), Before);
  a.edge_begin = Ranges(edges, S);
  CheckDeterminism(a.shift_targets, m.accept, edges, a.edge_begin);
  std::vector<BEdge> comps;
  if (merge) {
    comps = MergeComposites(edges, S, m.accept);
    std::sort(comps.begin(), comps.end(), Before);
  }
  a.stats.merged = static_cast<int64_t>(comps.size());
  a.composites = a.stats.merged;

  a.edges.reserve(edges.size());
  for (const BEdge& e : edges) a.edges.push_back(ToEdge(e));
  for (const BEdge& e : comps) a.composite_edges.push_back(ToEdge(e));
  for (const Circuit& c : cycles) a.cycle_list.push_back(CycleRec{c.states, c.closing});
  a.cycles = static_cast<int64_t>(cycles.size());
  return a;
}

void FinalizeAndCheck(Automaton* a) {
  std::vector<BEdge> edges, comps;
  for (const Edge& e : a->edges) edges.push_back(FromEdge(e));
  for (const Edge& e : a->composite_edges) comps.push_back(FromEdge(e));
  std::sort(edges.begin(), edges.end(), Before);
  std::sort(comps.begin(), comps.end(), Before);
  a->edge_begin = Ranges(edges, a->num_states);
  a->edges.clear();
  a->composite_edges.clear();
  for (const BEdge& e : edges) a->edges.push_back(ToEdge(e));
  for (const BEdge& e : comps) a->composite_edges.push_back(ToEdge(e));
  a->composites = static_cast<int64_t>(comps.size());
  a->cycles = static_cast<int64_t>(a->cycle_list.size());
  CheckDeterminism(a->shift_targets, a->accept_state, edges, a->edge_begin);
}

uint64_t GrammarHash(const std::string& normalized_text) { return Fnv1a(normalized_text); }

}  // namespace pre3
