// Pattern arity table, validation and JSON-lines I/O.
// Follows /root/reference/proj/include/ngdb/query.hpp:14-69 and SPEC.md:97-179.
#include "ngdb/query.hpp"

#include <cctype>
#include <fstream>
#include <sstream>

namespace ngdb {
namespace {

// name, anchors, relations, union, negation, eval nodes, train nodes.
// eval counts follow SPEC.md:130-131 (1p=3, 3i=8) and the DAG definitions in
// dag.cpp; training replaces Score by a fused Loss for non-union patterns and
// appends one Loss after UnionScore for union patterns (A-1).
constexpr PatternInfo kTable[kPatternCount] = {
    {"1p", 1, 1, false, false, 3, 3},   {"2p", 1, 2, false, false, 4, 4},
    {"3p", 1, 3, false, false, 5, 5},   {"2i", 2, 2, false, false, 6, 6},
    {"3i", 3, 3, false, false, 8, 8},   {"pi", 2, 3, false, false, 7, 7},
    {"ip", 2, 3, false, false, 7, 7},   {"2u", 2, 2, true, false, 7, 8},
    {"up", 2, 3, true, false, 9, 10},   {"2in", 2, 2, false, true, 7, 7},
    {"3in", 3, 3, false, true, 9, 9},   {"pin", 2, 3, false, true, 8, 8},
    {"pni", 2, 3, false, true, 8, 8},   {"inp", 2, 3, false, true, 8, 8},
};

constexpr std::array<Pattern, kPatternCount> kAll = {
    Pattern::P1, Pattern::P2,  Pattern::P3,  Pattern::I2,  Pattern::I3,
    Pattern::PI, Pattern::IP,  Pattern::U2,  Pattern::UP,  Pattern::IN2,
    Pattern::IN3, Pattern::PIN, Pattern::PNI, Pattern::INP};

void append_ids(std::string& out, const char* key, const std::vector<int32_t>& ids) {
  out += '"';
  out += key;
  out += "\":[";
  for (size_t i = 0; i < ids.size(); ++i) {
    if (i) out += ',';
    out += std::to_string(ids[i]);
  }
  out += ']';
}

// Minimal JSON reader for the flat record shape above.
struct Reader {
  const std::string& s;
  size_t i = 0;
  [[noreturn]] void fail(const char* what) const {
    throw ConfigError(std::string("malformed query record (") + what + ") at byte " +
                      std::to_string(i));
  }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  void expect(char c) {
    ws();
    if (i >= s.size() || s[i] != c) fail("unexpected character");
    ++i;
  }
  bool peek(char c) {
    ws();
    return i < s.size() && s[i] == c;
  }
  std::string str() {
    expect('"');
    std::string out;
    while (i < s.size() && s[i] != '"') out += s[i++];
    if (i >= s.size()) fail("unterminated string");
    ++i;
    return out;
  }
  std::vector<int32_t> ints() {
    std::vector<int32_t> out;
    expect('[');
    if (peek(']')) {
      ++i;
      return out;
    }
    for (;;) {
      ws();
      size_t start = i;
      if (i < s.size() && s[i] == '-') ++i;
      while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) ++i;
      if (start == i) fail("expected integer");
      out.push_back(static_cast<int32_t>(std::stol(s.substr(start, i - start))));
      ws();
      if (peek(',')) {
        ++i;
        continue;
      }
      expect(']');
      return out;
    }
  }
};

}  // namespace

const PatternInfo& pattern_info(Pattern p) { return kTable[static_cast<int>(p)]; }

const std::array<Pattern, kPatternCount>& all_patterns() { return kAll; }

Pattern parse_pattern(const std::string& name) {
  for (int i = 0; i < kPatternCount; ++i)
    if (name == kTable[i].name) return static_cast<Pattern>(i);
  throw UnsupportedPattern("unsupported pattern: " + name);
}

void QueryInstance::validate() const {
  const auto idx = static_cast<int>(pattern);
  if (idx < 0 || idx >= kPatternCount) throw UnsupportedPattern("pattern index out of range");
  const PatternInfo& info = kTable[idx];
  if (static_cast<int>(anchors.size()) != info.n_anchors ||
      static_cast<int>(relations.size()) != info.n_relations) {
    throw ArityMismatch(std::string(info.name) + " expects " + std::to_string(info.n_anchors) +
                        " anchors / " + std::to_string(info.n_relations) + " relations, got " +
                        std::to_string(anchors.size()) + " / " +
                        std::to_string(relations.size()));
  }
}

std::string to_jsonl(const QueryRecord& rec) {
  std::string out = "{\"pattern\":\"";
  out += pattern_info(rec.query.pattern).name;
  out += "\",";
  append_ids(out, "anchors", rec.query.anchors);
  out += ',';
  append_ids(out, "relations", rec.query.relations);
  out += ',';
  append_ids(out, "answers_obs", rec.answers_obs);
  out += ',';
  append_ids(out, "answers_miss", rec.answers_miss);
  out += '}';
  return out;
}

QueryRecord parse_jsonl(const std::string& line) {
  QueryRecord rec;
  Reader r{line};
  bool have_pattern = false;
  r.expect('{');
  if (!r.peek('}')) {
    for (;;) {
      const std::string key = r.str();
      r.expect(':');
      if (key == "pattern") {
        rec.query.pattern = parse_pattern(r.str());
        have_pattern = true;
      } else if (key == "anchors") {
        rec.query.anchors = r.ints();
      } else if (key == "relations") {
        rec.query.relations = r.ints();
      } else if (key == "answers_obs") {
        rec.answers_obs = r.ints();
      } else if (key == "answers_miss") {
        rec.answers_miss = r.ints();
      } else {
        r.fail("unknown key");
      }
      if (r.peek(',')) {
        ++r.i;
        continue;
      }
      break;
    }
  }
  r.expect('}');
  if (!have_pattern) r.fail("missing pattern");
  rec.query.validate();
  return rec;
}

std::vector<QueryRecord> load_query_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw MissingFile("cannot open " + path);
  std::vector<QueryRecord> out;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    out.push_back(parse_jsonl(line));
  }
  return out;
}

void save_query_file(const std::string& path, const std::vector<QueryRecord>& recs) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw MissingFile("cannot write " + path);
  for (const auto& r : recs) out << to_jsonl(r) << '\n';
}

}  // namespace ngdb
