// Native front end: graph JSON document -> operator-graph encoding + static
// features, bit-identical to the reference's Python front end (see
// include/dippm_host.h for the function map).  Host-only C++17; documents are
// independent, so a batch is spread over a thread pool.
//
// Reference semantics mirrored here (file:line in /root/reference/pkg/src/dippm):
//   JSON typing follows Python's json module: integers and floats are distinct
//   (isinstance(v, int) vs float), true/false are bools (excluded wherever the
//   reference says `not isinstance(v, bool)`), NaN/Infinity literals accepted,
//   duplicate object keys keep the last value.
//   parse_graph_json graph_ir.py:212-297 (check order preserved so the same
//   error class wins), _topological_order :300-323 (min-heap Kahn, inputs with
//   multiplicity), infer_shapes :357-499 (Python floor division), the
//   featurizer featurize.py:106-183 and compute_macs :204-253.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cerrno>
#include <queue>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/dippm_host.h"

namespace {

// ------------------------------------------------------------------ errors
struct Fail {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& m) { throw Fail{code, m}; }
std::string I(int64_t v) { return std::to_string(v); }

// ------------------------------------------------------------------ JSON
// A streaming parser specialised to the graph schema: one pass over the text
// records exactly what parse_graph_json inspects (value types, ids, names,
// inputs, known attributes, shapes) without building a document tree; every
// other value is skipped with full syntax validation, so a syntax error
// anywhere is a MalformedDocument exactly like json.loads failing first.
enum VT : uint8_t { V_NUL, V_BOOL, V_INT, V_FLT, V_STR, V_ARR, V_OBJ };

struct Scalar {
  uint8_t t = V_NUL;
  bool b = false;
  int64_t i = 0;
  double f = 0.0;
};

struct Cursor {
  const char* p;
  const char* e;
  int depth = 0;
  std::string tmp;  // decoded string with escapes
  Cursor(const char* b, const char* end) : p(b), e(end) {}
  [[noreturn]] void bad(const char* what) {
    fail(DIPPM_FEAT_MALFORMED_DOCUMENT, std::string("invalid JSON: ") + what);
  }
  inline void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool lit(const char* w, size_t n) {
    if ((size_t)(e - p) >= n && memcmp(p, w, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  static void put_utf8(std::string& out, uint32_t cp) {
    if (cp < 0x80) {
      out += (char)cp;
    } else if (cp < 0x800) {
      out += (char)(0xC0 | (cp >> 6));
      out += (char)(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += (char)(0xE0 | (cp >> 12));
      out += (char)(0x80 | ((cp >> 6) & 0x3F));
      out += (char)(0x80 | (cp & 0x3F));
    } else {
      out += (char)(0xF0 | (cp >> 18));
      out += (char)(0x80 | ((cp >> 12) & 0x3F));
      out += (char)(0x80 | ((cp >> 6) & 0x3F));
      out += (char)(0x80 | (cp & 0x3F));
    }
  }
  uint32_t hex4() {
    if (e - p < 4) bad("truncated \\u escape");
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= (uint32_t)(c - '0');
      else if (c >= 'a' && c <= 'f') v |= (uint32_t)(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= (uint32_t)(c - 'A' + 10);
      else bad("bad \\u escape");
    }
    return v;
  }
  // string at *p == '"'; returns a view valid until the next string() call
  std::string_view string() {
    const char* s0 = ++p;
    while (p < e) {  // fast path: no escapes
      const unsigned char c = (unsigned char)*p;
      if (c == '"') return std::string_view(s0, (size_t)(p++ - s0));
      if (c == '\\') break;
      if (c < 0x20) bad("control character in string");
      ++p;
    }
    tmp.assign(s0, (size_t)(p - s0));
    while (true) {
      if (p >= e) bad("unterminated string");
      const unsigned char c = (unsigned char)*p++;
      if (c == '"') break;
      if (c < 0x20) bad("control character in string");
      if (c != '\\') {
        tmp += (char)c;
        continue;
      }
      if (p >= e) bad("unterminated escape");
      const char x = *p++;
      switch (x) {
        case '"': tmp += '"'; break;
        case '\\': tmp += '\\'; break;
        case '/': tmp += '/'; break;
        case 'b': tmp += '\b'; break;
        case 'f': tmp += '\f'; break;
        case 'n': tmp += '\n'; break;
        case 'r': tmp += '\r'; break;
        case 't': tmp += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00 && e - p >= 6 && p[0] == '\\' && p[1] == 'u') {
            const char* save = p;
            p += 2;
            const uint32_t lo = hex4();
            if (lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            else p = save;
          }
          put_utf8(tmp, cp);
          break;
        }
        default: bad("bad escape");
      }
    }
    return std::string_view(tmp);
  }
  Scalar number() {
    const char* s0 = p;
    Scalar v;
    if (p < e && *p == '-') ++p;
    if (p < e && *p == 'I') {
      if (!lit("Infinity", 8)) bad("bad literal");
      v.t = V_FLT;
      v.f = -INFINITY;
      return v;
    }
    if (p >= e || !(*p >= '0' && *p <= '9')) bad("bad value");
    if (*p == '0') ++p;
    else
      while (p < e && *p >= '0' && *p <= '9') ++p;
    bool flt = false;
    if (p < e && *p == '.' && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
      flt = true;
      ++p;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      const char* q = p + 1;
      if (q < e && (*q == '+' || *q == '-')) ++q;
      if (q < e && *q >= '0' && *q <= '9') {
        flt = true;
        p = q;
        while (p < e && *p >= '0' && *p <= '9') ++p;
      }
    }
    const size_t n = (size_t)(p - s0);
    if (!flt && n <= 18) {  // fits int64 without overflow checks
      int64_t x = 0;
      const char* q = s0;
      const bool neg = *q == '-';
      if (neg) ++q;
      for (; q < p; ++q) x = x * 10 + (*q - '0');
      v.t = V_INT;
      v.i = neg ? -x : x;
      return v;
    }
    char buf[64];
    std::string big;
    const char* z;
    if (n < sizeof(buf)) {
      memcpy(buf, s0, n);
      buf[n] = 0;
      z = buf;
    } else {
      big.assign(s0, n);
      z = big.c_str();
    }
    if (flt) {
      v.t = V_FLT;
      v.f = strtod(z, nullptr);  // correctly rounded, like Python's float()
    } else {
      errno = 0;
      const long long x = strtoll(z, nullptr, 10);
      if (errno == ERANGE) fail(DIPPM_FEAT_UNSUPPORTED, "integer " + std::string(z) + " does not fit in 64 bits");
      v.t = V_INT;
      v.i = (int64_t)x;
    }
    return v;
  }
  // A scalar, or V_ARR / V_OBJ after skipping a container (validated).
  Scalar value() {
    ws();
    if (p >= e) bad("unexpected end");
    Scalar v;
    switch (*p) {
      case '{': skip_container(); v.t = V_OBJ; return v;
      case '[': skip_container(); v.t = V_ARR; return v;
      case '"': string(); v.t = V_STR; return v;
      case 't': if (lit("true", 4)) { v.t = V_BOOL; v.b = true; return v; } break;
      case 'f': if (lit("false", 5)) { v.t = V_BOOL; return v; } break;
      case 'n': if (lit("null", 4)) return v; break;
      case 'N': if (lit("NaN", 3)) { v.t = V_FLT; v.f = NAN; return v; } break;
      case 'I': if (lit("Infinity", 8)) { v.t = V_FLT; v.f = INFINITY; return v; } break;
      default: return number();
    }
    bad("bad literal");
  }
  void skip_container() {
    if (++depth > 512) bad("nesting too deep");
    const char open = *p++;
    const char close = open == '{' ? '}' : ']';
    ws();
    if (p < e && *p == close) {
      ++p;
      --depth;
      return;
    }
    while (true) {
      if (open == '{') {
        ws();
        if (p >= e || *p != '"') bad("expected key");
        string();
        ws();
        if (p >= e || *p != ':') bad("expected ':'");
        ++p;
      }
      value();
      ws();
      if (p < e && *p == ',') {
        ++p;
        continue;
      }
      if (p < e && *p == close) {
        ++p;
        break;
      }
      bad("expected ',' or closing bracket");
    }
    --depth;
  }
  // Iterate an object's members: f(key) must consume the value and must not
  // use `key` after parsing any string of that value.
  template <class F>
  void object(F&& f) {
    ++p;
    ws();
    if (p < e && *p == '}') {
      ++p;
      return;
    }
    while (true) {
      ws();
      if (p >= e || *p != '"') bad("expected key");
      const std::string_view key = string();  // valid until f parses another string
      ws();
      if (p >= e || *p != ':') bad("expected ':'");
      ++p;
      ws();
      f(key);
      ws();
      if (p < e && *p == ',') {
        ++p;
        continue;
      }
      if (p < e && *p == '}') {
        ++p;
        return;
      }
      bad("expected ',' or '}'");
    }
  }
  // Iterate an array's elements: f() must consume each element.
  template <class F>
  void array(F&& f) {
    ++p;
    ws();
    if (p < e && *p == ']') {
      ++p;
      return;
    }
    while (true) {
      ws();
      f();
      ws();
      if (p < e && *p == ',') {
        ++p;
        continue;
      }
      if (p < e && *p == ']') {
        ++p;
        return;
      }
      bad("expected ',' or ']'");
    }
  }
  bool peek(char c) {
    ws();
    return p < e && *p == c;
  }
};

// ------------------------------------------------------------------ IR
// Operator vocabulary, definition order = one-hot order (graph_ir.py:53-79).
const char* const kKinds[16] = {"conv2d",   "conv2d_transpose", "dense",           "batch_matmul", "relu",    "add",
                                "multiply", "maxpool2d",        "avgpool2d",       "global_avgpool2d", "batchnorm",
                                "softmax",  "reshape",          "concat",          "layernorm",    "other"};
enum Kind {
  CONV2D = 0, CONV2D_T, DENSE, BMM, RELU, ADD, MUL, MAXPOOL, AVGPOOL, GAVGPOOL, BATCHNORM, SOFTMAX, RESHAPE, CONCAT,
  LAYERNORM, OTHER
};
// KNOWN_ATTRIBUTES order (graph_ir.py:84-97) = feature slots 16..27
const char* const kAttrs[12] = {"kernel_h",   "kernel_w",   "stride_h", "stride_w",     "pad_h",    "pad_w",
                                "dilation_h", "dilation_w", "groups",   "out_features", "has_bias", "epsilon"};
enum Attr { KH = 0, KW, SH, SW, PH, PW, DH, DW, GROUPS, OUTF, HAS_BIAS, EPS };
const char* const kNonOperator[10] = {"const", "constant", "var", "variable", "param", "parameter", "input", "tuple",
                                      "tuple_get_item", "tuplegetitem"};  // graph_ir.py:101-114

// classify an operator tail (lower-cased): one-hot kind and is_operator
void classify(std::string_view tail, int& kind, bool& is_op) {
  static const std::string_view kinds[16] = {kKinds[0], kKinds[1], kKinds[2],  kKinds[3],  kKinds[4],  kKinds[5],
                                             kKinds[6], kKinds[7], kKinds[8],  kKinds[9],  kKinds[10], kKinds[11],
                                             kKinds[12], kKinds[13], kKinds[14], kKinds[15]};
  static const std::string_view non_op[10] = {kNonOperator[0], kNonOperator[1], kNonOperator[2], kNonOperator[3],
                                              kNonOperator[4], kNonOperator[5], kNonOperator[6], kNonOperator[7],
                                              kNonOperator[8], kNonOperator[9]};
  kind = OTHER;
  for (int q = 0; q < 16; ++q)
    if (tail == kinds[q]) kind = q;
  is_op = true;
  for (const std::string_view& w : non_op)
    if (tail == w) is_op = false;
}

std::string op_tail(const std::string& raw) {  // name.strip().lower().rsplit(".", 1)[-1]
  size_t a = 0, b = raw.size();
  auto sp = [](unsigned char c) { return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f); };
  while (a < b && sp((unsigned char)raw[a])) ++a;
  while (b > a && sp((unsigned char)raw[b - 1])) --b;
  std::string t = raw.substr(a, b - a);
  for (auto& ch : t)
    if (ch >= 'A' && ch <= 'Z') ch = (char)(ch - 'A' + 'a');
  size_t dot = t.rfind('.');
  return dot == std::string::npos ? t : t.substr(dot + 1);
}

struct Node {
  std::string raw;
  int kind = OTHER;
  bool is_op = true;
  bool has_attr[12] = {};
  double attr[12] = {};      // float(value)
  bool attr_int[12] = {};    // value was a JSON integer (int() is then exact)
  int64_t attr_i[12] = {};
  bool has_shape = false;
  std::vector<int64_t> shape;
  std::vector<int64_t> inputs;
  // this <- src for the fields the graph uses; the buffers are exchanged, not copied (src is
  // reset before its next use)
  void take(Node& src) {
    raw.swap(src.raw);
    shape.swap(src.shape);
    inputs.swap(src.inputs);
    kind = src.kind;
    is_op = src.is_op;
    has_shape = src.has_shape;
    for (int a = 0; a < 12; ++a) {
      has_attr[a] = src.has_attr[a];
      attr[a] = src.attr[a];
      attr_int[a] = src.attr_int[a];
      attr_i[a] = src.attr_i[a];
    }
  }
  void reset() {  // a fresh node, keeping the vectors' capacity
    raw.clear();
    kind = OTHER;
    is_op = true;
    for (int a = 0; a < 12; ++a) {
      has_attr[a] = attr_int[a] = false;
      attr[a] = 0.0;
      attr_i[a] = 0;
    }
    has_shape = false;
    shape.clear();
    inputs.clear();
  }
};

struct Graph {
  std::vector<Node> nodes;
  std::vector<int64_t> outputs;
  int64_t batch = 1;
  std::string name;
};

double attr_f(const Node& n, int a) { return n.has_attr[a] ? n.attr[a] : 0.0; }
// int(node.attr(name)): exact for integers, truncation toward zero for floats
int64_t attr_int(const Node& n, int a) {
  if (!n.has_attr[a]) return 0;
  if (n.attr_int[a]) return n.attr_i[a];
  double v = n.attr[a];
  if (std::isnan(v)) fail(DIPPM_FEAT_VALUE_ERROR, "cannot convert float NaN to integer");
  if (std::isinf(v)) fail(DIPPM_FEAT_VALUE_ERROR, "cannot convert float infinity to integer");
  double t = std::trunc(v);
  if (t >= 9.2233720368547758e18 || t < -9.2233720368547758e18) fail(DIPPM_FEAT_UNSUPPORTED, "attribute too large");
  return (int64_t)t;
}

int64_t floordiv(int64_t a, int64_t b) {  // Python //
  if (b == 0) fail(DIPPM_FEAT_VALUE_ERROR, "integer division or modulo by zero");
  int64_t q = a / b, r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) --q;
  return q;
}

std::string shape_str(const std::vector<int64_t>& s) {
  std::string o = "[";
  for (size_t k = 0; k < s.size(); ++k) o += (k ? ", " : "") + I(s[k]);
  return o + "]";
}

void check_shape(const std::vector<int64_t>& s, int64_t id) {  // graph_ir.py:200-205
  if (s.size() < 1 || s.size() > 4)
    fail(DIPPM_FEAT_BAD_SHAPE, "node " + I(id) + ": shape rank " + I((int64_t)s.size()) + " outside [1, 4]");
  for (int64_t d : s)
    if (d < 1) fail(DIPPM_FEAT_BAD_SHAPE, "node " + I(id) + ": shape entry " + I(d) + " is not a positive integer");
}

// What one node entry of the document holds (last duplicate key wins).
struct RawNode {
  bool is_obj = false;
  bool has_id = false;
  Scalar id;
  bool has_op = false;
  uint8_t op_t = V_NUL;
  std::string op;
  bool has_inputs = false;
  uint8_t inputs_t = V_NUL;
  bool inputs_ok = true;  // every element an int (not bool)
  std::vector<int64_t> inputs;
  bool has_attrs = false;
  uint8_t attrs_t = V_NUL;
  bool has_known[12] = {};                            // KNOWN_ATTRIBUTES, last duplicate wins
  Scalar known[12];
  std::vector<std::pair<std::string, Scalar>> attrs;  // other names (only their types matter)
  bool has_shape = false;
  uint8_t shape_t = V_NUL;
  std::vector<Scalar> shape;
  void reset() {  // back to the parsed-nothing state, keeping the vectors' capacity
    is_obj = has_id = has_op = has_inputs = has_attrs = has_shape = false;
    id = Scalar();
    op_t = inputs_t = attrs_t = shape_t = V_NUL;
    op.clear();
    inputs_ok = true;
    inputs.clear();
    for (bool& h : has_known) h = false;
    attrs.clear();
    shape.clear();
  }
};

// Per-thread pool of node entries: documents are parsed back to back on a worker thread, so
// the entries (and their small vectors) are reused instead of reallocated per node.
struct RawPool {
  std::vector<RawNode> v;
  size_t n = 0;
  RawNode& next() {
    if (n == v.size()) v.emplace_back();
    RawNode& r = v[n++];
    r.reset();
    return r;
  }
  RawNode* begin() { return v.data(); }
  RawNode* end() { return v.data() + n; }
  size_t size() const { return n; }
  bool empty() const { return n == 0; }
};

void read_node(Cursor& c, RawNode& r) {
  r.is_obj = true;
  c.object([&](std::string_view key) {
    if (key == "id") {
      r.has_id = true;
      r.id = c.value();
    } else if (key == "op") {
      r.has_op = true;
      if (c.peek('"')) {
        r.op_t = V_STR;
        r.op = std::string(c.string());
      } else {
        r.op_t = c.value().t;
        r.op.clear();
      }
    } else if (key == "inputs") {
      r.has_inputs = true;
      r.inputs.clear();
      r.inputs_ok = true;
      if (c.peek('[')) {
        r.inputs_t = V_ARR;
        c.array([&] {
          const Scalar v = c.value();
          if (v.t == V_INT) r.inputs.push_back(v.i);
          else r.inputs_ok = false;
        });
      } else {
        r.inputs_t = c.value().t;
      }
    } else if (key == "attrs") {
      r.has_attrs = true;
      r.attrs.clear();
      for (bool& h : r.has_known) h = false;
      if (c.peek('{')) {
        r.attrs_t = V_OBJ;
        c.object([&](std::string_view k) {
          static const std::string_view names[12] = {kAttrs[0], kAttrs[1], kAttrs[2], kAttrs[3],
                                                     kAttrs[4], kAttrs[5], kAttrs[6], kAttrs[7],
                                                     kAttrs[8], kAttrs[9], kAttrs[10], kAttrs[11]};
          int slot = -1;
          for (int a = 0; a < 12 && slot < 0; ++a)
            if (k == names[a]) slot = a;
          if (slot >= 0) {
            r.known[slot] = c.value();
            r.has_known[slot] = true;
            return;
          }
          std::string key(k);  // copy before the value may overwrite the view
          const Scalar v = c.value();
          for (auto& kv : r.attrs)
            if (kv.first == key) {
              kv.second = v;
              return;
            }
          r.attrs.emplace_back(std::move(key), v);
        });
      } else {
        r.attrs_t = c.value().t;
      }
    } else if (key == "out_shape") {
      r.has_shape = true;
      r.shape.clear();
      if (c.peek('[')) {
        r.shape_t = V_ARR;
        c.array([&] { r.shape.push_back(c.value()); });
      } else {
        r.shape_t = c.value().t;
      }
    } else {
      c.value();
    }
  });
}

// node id -> entry index: a direct table when the ids are dense (the usual 0..n-1 numbering),
// else a hash map.
struct IdIndex {
  std::vector<int32_t> table;
  std::unordered_map<int64_t, size_t> map;
  bool dense = true;
  explicit IdIndex(RawPool& raw) {
    int64_t hi = -1;
    for (const RawNode& r : raw)
      if (r.is_obj && r.has_id && r.id.t == V_INT) hi = std::max(hi, r.id.i);
    dense = hi < (int64_t)raw.size() * 4 + 64;
    if (dense) table.assign((size_t)(hi + 1), -1);
    else map.reserve(raw.size() * 2);
  }
  int64_t find(int64_t id) const {
    if (dense) return (id >= 0 && id < (int64_t)table.size()) ? table[(size_t)id] : -1;
    auto it = map.find(id);
    return it == map.end() ? -1 : (int64_t)it->second;
  }
  size_t at(int64_t id) const { return (size_t)find(id); }  // id known to exist
  void set(int64_t id, size_t k) {
    if (dense) table[(size_t)id] = (int32_t)k;
    else map[id] = k;
  }
};

// parse_graph_json graph_ir.py:212-297.  g is the caller's (per-thread, reused) graph.
void parse_graph(const char* text, int64_t len, Graph& g) {
  Cursor c{text, text + len};
  bool has_nodes = false, nodes_arr = false, has_outputs = false, outputs_arr = false, has_batch = false,
       has_name = false;
  static thread_local RawPool raw;
  raw.n = 0;
  std::vector<Scalar> outputs;
  Scalar batch, name_v;
  std::string name;
  c.ws();
  if (!c.peek('{')) {
    c.value();  // a valid non-object document (or a syntax error)
    c.ws();
    if (c.p != c.e) c.bad("extra data");
    fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "top-level value must be an object");
  }
  c.object([&](std::string_view key) {
    if (key == "nodes") {
      has_nodes = true;
      raw.n = 0;
      nodes_arr = c.peek('[');
      if (nodes_arr) {
        c.array([&] {
          RawNode& r = raw.next();
          if (c.peek('{')) read_node(c, r);
          else c.value();
        });
      } else {
        c.value();
      }
    } else if (key == "outputs") {
      has_outputs = true;
      outputs.clear();
      outputs_arr = c.peek('[');
      if (outputs_arr) c.array([&] { outputs.push_back(c.value()); });
      else c.value();
    } else if (key == "batch") {
      has_batch = true;
      batch = c.value();
    } else if (key == "name") {
      has_name = true;
      if (c.peek('"')) {
        name_v.t = V_STR;
        name = std::string(c.string());
      } else {
        name_v = c.value();
      }
    } else {
      c.value();
    }
  });
  c.ws();
  if (c.p != c.e) c.bad("extra data");

  if (!has_nodes || !nodes_arr || raw.empty())
    fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "\"nodes\" must be a non-empty list");
  bool ok = has_outputs && outputs_arr && !outputs.empty();
  if (ok)
    for (const Scalar& o : outputs)
      if (!(o.t == V_INT || o.t == V_BOOL)) ok = false;  // isinstance(o, int): bool is an int
  if (!ok) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "\"outputs\" must be a non-empty list of node ids");
  if (!has_batch || batch.t != V_INT || batch.i < 1)
    fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "\"batch\" must be a positive integer");
  if (has_name && name_v.t != V_STR) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "\"name\" must be a string");

  IdIndex by_id(raw);
  std::vector<int64_t> order_doc;
  order_doc.reserve(raw.size());
  // document-order entries, a per-thread pool swapped with g.nodes below (capacity reused)
  static thread_local std::vector<Node> entries;
  if (entries.size() < raw.size()) entries.resize(raw.size());
  size_t ne = 0;
  for (RawNode& r : raw) {
    if (!r.is_obj) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "every node must be an object");
    if (!r.has_id || r.id.t != V_INT || r.id.i < 0)
      fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "node id must be a non-negative integer");
    const int64_t nid = r.id.i;
    if (by_id.find(nid) >= 0) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "duplicate node id " + I(nid));
    if (!r.has_op || r.op_t != V_STR || r.op.empty())
      fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "node " + I(nid) + ": missing operator name");
    Node& n = entries[ne];
    n.reset();
    n.raw = r.op;
    if (r.has_inputs) {
      if (r.inputs_t != V_ARR || !r.inputs_ok)
        fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "node " + I(nid) + ": inputs must be a list of node ids");
      n.inputs = r.inputs;
    }
    if (r.has_attrs) {
      bool good = r.attrs_t == V_OBJ;
      if (good)
        for (const auto& kv : r.attrs)
          if (kv.second.t != V_INT && kv.second.t != V_FLT) good = false;
      for (int a = 0; a < 12; ++a)
        if (r.has_known[a] && r.known[a].t != V_INT && r.known[a].t != V_FLT) good = false;
      if (!good) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "node " + I(nid) + ": attrs must map names to numbers");
      for (int a = 0; a < 12; ++a)
        if (r.has_known[a]) {
          const Scalar& v = r.known[a];
          n.has_attr[a] = true;
          n.attr_int[a] = v.t == V_INT;
          n.attr_i[a] = v.i;
          n.attr[a] = v.t == V_INT ? (double)v.i : v.f;
        }
    }
    if (r.has_shape && r.shape_t != V_NUL) {
      if (r.shape_t != V_ARR) fail(DIPPM_FEAT_BAD_SHAPE, "node " + I(nid) + ": out_shape must be a list");
      if (r.shape.size() < 1 || r.shape.size() > 4)
        fail(DIPPM_FEAT_BAD_SHAPE, "node " + I(nid) + ": shape rank " + I((int64_t)r.shape.size()) + " outside [1, 4]");
      for (const Scalar& d : r.shape) {
        if (d.t != V_INT || d.i < 1)
          fail(DIPPM_FEAT_BAD_SHAPE, "node " + I(nid) + ": shape entry is not a positive integer");
        n.shape.push_back(d.i);
      }
      n.has_shape = true;
    }
    by_id.set(nid, ne);
    order_doc.push_back(nid);
    ++ne;
  }
  for (size_t k = 0; k < ne; ++k)
    for (int64_t src : entries[k].inputs)
      if (by_id.find(src) < 0)
        fail(DIPPM_FEAT_DANGLING_REFERENCE, "node " + I(order_doc[k]) + " references missing input " + I(src));
  for (const Scalar& o : outputs) {
    const int64_t oid = o.t == V_BOOL ? (int64_t)o.b : o.i;
    if (by_id.find(oid) < 0) fail(DIPPM_FEAT_DANGLING_REFERENCE, "output id " + I(oid) + " does not exist");
  }
  // _topological_order: Kahn over a min-heap of original ids, inputs counted with multiplicity.
  // Ids are renamed to entry indices for the bookkeeping; the heap orders by original id.
  const size_t M = ne;
  std::vector<int64_t> pending(M), cptr(M + 1, 0);
  std::vector<size_t> cons;
  for (size_t k = 0; k < M; ++k) {
    pending[k] = (int64_t)entries[k].inputs.size();
    for (int64_t src : entries[k].inputs) ++cptr[by_id.at(src) + 1];
  }
  for (size_t k = 0; k < M; ++k) cptr[k + 1] += cptr[k];
  cons.resize((size_t)cptr[M]);
  {
    std::vector<int64_t> fillp(cptr.begin(), cptr.end() - 1);
    for (size_t k = 0; k < M; ++k)  // consumers in document order, like the reference's dict
      for (int64_t src : entries[k].inputs) cons[(size_t)fillp[by_id.at(src)]++] = k;
  }
  std::priority_queue<std::pair<int64_t, size_t>, std::vector<std::pair<int64_t, size_t>>, std::greater<>> heap;
  for (size_t k = 0; k < M; ++k)
    if (pending[k] == 0) heap.push({order_doc[k], k});
  std::vector<size_t> order;
  order.reserve(M);
  while (!heap.empty()) {
    const size_t k = heap.top().second;
    heap.pop();
    order.push_back(k);
    for (int64_t j = cptr[k]; j < cptr[k + 1]; ++j) {
      const size_t cidx = cons[(size_t)j];
      if (--pending[cidx] == 0) heap.push({order_doc[cidx], cidx});
    }
  }
  if (order.size() != M) {
    std::vector<char> done(M, 0);
    for (size_t k : order) done[k] = 1;
    std::vector<int64_t> stuck;
    for (size_t k = 0; k < M; ++k)
      if (!done[k]) stuck.push_back(order_doc[k]);
    std::sort(stuck.begin(), stuck.end());
    fail(DIPPM_FEAT_CYCLIC_GRAPH, "nodes " + shape_str(stuck) + " form a dependency cycle");
  }
  std::vector<int64_t> remap(M);
  for (size_t k = 0; k < M; ++k) remap[order[k]] = (int64_t)k;
  g.batch = batch.i;
  g.name = std::move(name);
  g.nodes.resize(M);
  for (size_t i = 0; i < M; ++i) {
    g.nodes[i].take(entries[order[i]]);  // entries keeps the previous graph's buffers
    Node& n = g.nodes[i];
    for (auto& x : n.inputs) x = remap[by_id.at(x)];
    classify(op_tail(n.raw), n.kind, n.is_op);
  }
  g.outputs.clear();
  for (const Scalar& o : outputs) g.outputs.push_back(remap[by_id.at(o.t == V_BOOL ? (int64_t)o.b : o.i)]);
}

int64_t numel(const std::vector<int64_t>& s) {
  __int128 n = 1;
  for (int64_t d : s) n *= d;
  if (n > INT64_MAX) fail(DIPPM_FEAT_UNSUPPORTED, "tensor size beyond 64 bits");
  return (int64_t)n;
}

int64_t conv_spatial(int64_t size, int64_t k, int64_t s, int64_t pad, int64_t dil) {
  return floordiv(size + 2 * pad - dil * (k - 1) - 1, s) + 1;
}

// _infer_node_shape graph_ir.py:384-493
using Shapes = std::vector<const std::vector<int64_t>*>;
std::vector<int64_t> infer_node(const Node& n, int64_t id, const Shapes& in) {
  const auto nid = [id] { return I(id); };  // built only on failure
  if (n.inputs.empty()) {
    if (!n.has_shape) fail(DIPPM_FEAT_UNDERSPECIFIED, "source node " + nid() + " (" + n.raw + ") declares no out_shape");
    return n.shape;
  }
  const int k = n.kind;
  const auto& first = *in[0];
  if (k == CONV2D || k == CONV2D_T) {
    if (first.size() != 4)
      fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid() + ": " + kKinds[k] + " input must be rank 4, got " + shape_str(first));
    const int64_t kh = attr_int(n, KH), kw = attr_int(n, KW);
    if (kh < 1 || kw < 1) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid() + ": " + kKinds[k] + " kernel size missing");
    int64_t sh = attr_int(n, SH), sw = attr_int(n, SW);
    if (!sh) sh = 1;
    if (!sw) sw = 1;
    const int64_t ph = attr_int(n, PH), pw = attr_int(n, PW);
    int64_t dh = attr_int(n, DH), dw = attr_int(n, DW);
    if (!dh) dh = 1;
    if (!dw) dw = 1;
    int64_t out_c = attr_int(n, OUTF);
    if (out_c < 1) {
      if (n.has_shape && n.shape.size() == 4) out_c = n.shape[1];
      else fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid() + ": " + kKinds[k] + " output channels missing");
    }
    const int64_t nn = first[0], h = first[2], w = first[3];
    if (k == CONV2D) return {nn, out_c, conv_spatial(h, kh, sh, ph, dh), conv_spatial(w, kw, sw, pw, dw)};
    return {nn, out_c, (h - 1) * sh - 2 * ph + dh * (kh - 1) + 1, (w - 1) * sw - 2 * pw + dw * (kw - 1) + 1};
  }
  if (k == MAXPOOL || k == AVGPOOL) {
    if (first.size() != 4)
      fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid() + ": " + kKinds[k] + " input must be rank 4, got " + shape_str(first));
    const int64_t kh = attr_int(n, KH), kw = attr_int(n, KW);
    if (kh < 1 || kw < 1) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid() + ": pool kernel size missing");
    int64_t sh = attr_int(n, SH), sw = attr_int(n, SW);
    if (!sh) sh = kh;
    if (!sw) sw = kw;
    const int64_t ph = attr_int(n, PH), pw = attr_int(n, PW);
    int64_t dh = attr_int(n, DH), dw = attr_int(n, DW);
    if (!dh) dh = 1;
    if (!dw) dw = 1;
    return {first[0], first[1], conv_spatial(first[2], kh, sh, ph, dh), conv_spatial(first[3], kw, sw, pw, dw)};
  }
  if (k == GAVGPOOL) {
    if (first.size() != 4)
      fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid() + ": global pool input must be rank 4, got " + shape_str(first));
    return {first[0], first[1], 1, 1};
  }
  if (k == DENSE) {
    const int64_t of = attr_int(n, OUTF);
    if (of < 1) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid() + ": dense out_features missing");
    std::vector<int64_t> r(first.begin(), first.end() - 1);
    r.push_back(of);
    return r;
  }
  if (k == BMM) {
    if (in.size() != 2) fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid() + ": batch_matmul needs exactly 2 inputs");
    const auto &a = *in[0], &b = *in[1];
    if (a.size() != 3 || b.size() != 3)
      fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid() + ": batch_matmul inputs must be rank 3");
    if (a[0] != b[0] || a[2] != b[1]) fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid() + ": batch_matmul shapes do not compose");
    return {a[0], a[1], b[2]};
  }
  if (k == ADD || k == MUL) {
    for (size_t j = 1; j < in.size(); ++j)
      if (*in[j] != first) fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid() + ": elementwise inputs differ");
    return first;
  }
  if (k == CONCAT) {
    if (first.size() < 2) fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid() + ": concat inputs must have rank >= 2");
    int64_t ch = 0;
    for (const auto* sp : in) {
      const auto& s = *sp;
      bool same = s.size() == first.size() && s[0] == first[0];
      for (size_t d = 2; same && d < s.size(); ++d) same = s[d] == first[d];
      if (!same) fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid() + ": concat inputs differ outside channel dim");
      ch += s[1];
    }
    std::vector<int64_t> r = {first[0], ch};
    r.insert(r.end(), first.begin() + 2, first.end());
    return r;
  }
  if (k == RESHAPE) {
    const int64_t total = numel(first);
    if (n.has_shape && numel(n.shape) == total) return n.shape;
    if (first.size() < 2) return first;
    return {first[0], floordiv(total, first[0])};
  }
  if (k == RELU || k == SOFTMAX || k == BATCHNORM || k == LAYERNORM) return first;
  if (n.has_shape) return n.shape;  // OTHER: trust a declared shape, else pass through
  return first;
}

void infer_shapes(Graph& g) {  // graph_ir.py:357-381 (validation already holds after parsing)
  // Nodes are in topological order and inputs precede their consumers, so a node's inferred
  // shape can replace its declared one as soon as it is known: later nodes only read the
  // inferred shapes of their inputs (the reference's `shapes` dict) and their own declared
  // shape.  A failure discards the whole graph.
  Shapes in;
  for (size_t k = 0; k < g.nodes.size(); ++k) {
    Node& n = g.nodes[k];
    in.clear();
    for (int64_t i : n.inputs) in.push_back(&g.nodes[i].shape);
    std::vector<int64_t> s = infer_node(n, (int64_t)k, in);
    check_shape(s, (int64_t)k);
    n.shape = std::move(s);
    n.has_shape = true;
  }
}

void with_batch_size(Graph& g, int64_t b) {  // graph_ir.py:502-529
  if (b < 1) fail(DIPPM_FEAT_INVALID_SPEC, "batch size must be positive, got " + I(b));
  const int64_t old = g.batch;
  for (Node& n : g.nodes) {
    if (!n.inputs.empty() || !n.has_shape) {
      n.has_shape = false;
      n.shape.clear();
      continue;
    }
    if (n.shape.size() >= 2 && n.shape[0] == old) n.shape[0] = b;
  }
  g.batch = b;
  infer_shapes(g);
}

struct Result {
  int status = DIPPM_FEAT_OK;
  std::string msg, name;
  int64_t n = 0;
  std::vector<std::pair<int64_t, int64_t>> edges;
  std::vector<double> x;
  int64_t fs[5] = {0, 0, 0, 0, 0};
};

// operator_graph featurize.py:106-163
void operator_graph(const Graph& g, std::vector<int64_t>& order, std::vector<std::pair<int64_t, int64_t>>& edges) {
  const size_t N = g.nodes.size();
  bool any = false;
  for (const Node& n : g.nodes) any |= n.is_op;
  if (!any) fail(DIPPM_FEAT_EMPTY_GRAPH, "graph '" + g.name + "' has no operator nodes");
  // producers of node v = prod[pptr[v] .. pptr[v+1]) (deduplicated, input order kept)
  std::vector<int64_t> prod, pptr(N + 1, 0);
  prod.reserve(N * 2);
  for (size_t v = 0; v < N; ++v) {
    const size_t s0 = prod.size();
    auto add = [&](int64_t c) {
      for (size_t j = s0; j < prod.size(); ++j)
        if (prod[j] == c) return;
      prod.push_back(c);
    };
    for (int64_t src : g.nodes[v].inputs) {
      if (g.nodes[src].is_op) add(src);
      else
        for (int64_t j = pptr[src]; j < pptr[src + 1]; ++j) add(prod[(size_t)j]);
    }
    pptr[v + 1] = (int64_t)prod.size();
  }
  struct Span {
    const int64_t* b;
    const int64_t* e;
    const int64_t* begin() const { return b; }
    const int64_t* end() const { return e; }
  };
  auto producers = [&](int64_t v) { return Span{prod.data() + pptr[v], prod.data() + pptr[v + 1]}; };
  std::vector<char> visited(N, 0);
  std::vector<std::pair<int64_t, bool>> stack;
  auto visit = [&](int64_t root) {
    stack.assign(1, {root, false});
    while (!stack.empty()) {
      auto [nid, expanded] = stack.back();
      stack.pop_back();
      if (expanded) {
        order.push_back(nid);
        continue;
      }
      if (visited[nid]) continue;
      visited[nid] = 1;
      stack.push_back({nid, true});
      const Span pr = producers(nid);
      for (const int64_t* it = pr.e; it != pr.b;) {
        --it;
        if (!visited[*it]) stack.push_back({*it, false});
      }
    }
  };
  for (int64_t out : g.outputs) {
    if (g.nodes[out].is_op) {
      if (!visited[out]) visit(out);
    } else {
      for (int64_t r : producers(out))
        if (!visited[r]) visit(r);
    }
  }
  for (size_t v = 0; v < N; ++v)
    if (g.nodes[v].is_op && !visited[v]) visit((int64_t)v);
  std::vector<int64_t> position(N, -1);
  for (size_t i = 0; i < order.size(); ++i) position[order[i]] = (int64_t)i;
  // The reference filters through an `emitted` set; it never fires: every node occurs once in
  // `order` and its producer list is already deduplicated, so (src, nid) pairs are unique.
  edges.reserve(prod.size());
  for (int64_t nid : order)
    for (int64_t src : producers(nid)) edges.push_back({position[src], position[nid]});
}

// encode_node featurize.py:166-183
void encode_node(const Node& n, double* vec) {
  for (int k = 0; k < 32; ++k) vec[k] = 0.0;
  vec[n.kind] = 1.0;
  for (int a = 0; a < 12; ++a) {
    const double v = attr_f(n, a);
    if (a == HAS_BIAS) vec[16 + a] = (v != 0.0 || std::isnan(v)) ? 1.0 : 0.0;  // truthiness of the value
    else if (a == EPS) vec[16 + a] = v;
    else vec[16 + a] = std::log1p((0.0 > v) ? 0.0 : v);  // max(value, 0.0) keeps NaN and -0.0 like Python
  }
  for (size_t ax = 0; ax < n.shape.size(); ++ax) vec[28 + ax] = std::log1p((double)n.shape[ax]);
}

int64_t checked(__int128 v) {
  if (v > INT64_MAX || v < INT64_MIN) fail(DIPPM_FEAT_UNSUPPORTED, "MAC count beyond 64 bits");
  return (int64_t)v;
}

// compute_macs / _node_macs featurize.py:204-253
int64_t compute_macs(const Graph& g) {
  __int128 total = 0;
  for (size_t k = 0; k < g.nodes.size(); ++k) {
    const Node& n = g.nodes[k];
    if (n.kind != CONV2D && n.kind != CONV2D_T && n.kind != DENSE && n.kind != BMM) continue;
    const auto nid = [k] { return I((int64_t)k); };
    if (n.inputs.empty()) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid() + ": input shape unavailable");
    const auto& in = g.nodes[n.inputs[0]].shape;
    const auto& out = n.shape;
    if (n.kind == DENSE) {
      __int128 lead = 1;
      for (size_t d = 0; d + 1 < out.size(); ++d) lead *= out[d];
      total += lead * in.back() * out.back();
    } else if (n.kind == BMM) {
      if (out.size() < 3 || in.size() < 3) fail(DIPPM_FEAT_VALUE_ERROR, "node " + nid() + ": list index out of range");
      total += (__int128)out[0] * out[1] * out[2] * in[2];
    } else {
      const int64_t kh = attr_int(n, KH), kw = attr_int(n, KW);
      if (kh < 1 || kw < 1) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid() + ": kernel size missing");
      int64_t groups = attr_int(n, GROUPS);
      if (!groups) groups = 1;
      if (in.size() != 4 || out.size() != 4) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid() + ": conv shapes must be rank 4");
      if (n.kind == CONV2D)
        total += (__int128)out[0] * out[1] * out[2] * out[3] * floordiv(in[1], groups) * kh * kw;
      else
        total += (__int128)in[0] * in[1] * in[2] * in[3] * floordiv(out[1], groups) * kh * kw;
    }
    checked(total);
  }
  return checked(total);
}

void featurize_one(const char* doc, int64_t len, int64_t batch_override, Result& r) {
  try {
    static thread_local Graph g;
    parse_graph(doc, len, g);
    bool missing = false;
    for (const Node& n : g.nodes) missing |= !n.has_shape;
    if (missing) infer_shapes(g);
    if (batch_override != 0) with_batch_size(g, batch_override);
    std::vector<int64_t> order;
    operator_graph(g, order, r.edges);
    r.n = (int64_t)order.size();
    r.x.assign((size_t)r.n * 32, 0.0);
    for (size_t i = 0; i < order.size(); ++i) {
      const Node& n = g.nodes[order[i]];
      encode_node(n, &r.x[i * 32]);
    }
    r.fs[0] = compute_macs(g);
    r.fs[1] = g.batch;
    for (const Node& n : g.nodes) {
      r.fs[2] += n.kind == CONV2D;
      r.fs[3] += n.kind == DENSE;
      r.fs[4] += n.kind == RELU;
    }
    r.name = g.name;
  } catch (const Fail& f) {
    r = Result();
    r.status = f.code;
    r.msg = f.msg;
  } catch (const std::bad_alloc&) {
    r = Result();
    r.status = DIPPM_FEAT_UNSUPPORTED;
    r.msg = "out of memory";
  }
}

}  // namespace

struct dippm_feat_batch {
  std::vector<Result> res;
};

extern "C" {

int32_t dippm_host_abi_version(void) { return DIPPM_HOST_ABI_VERSION; }

dippm_feat_batch* dippm_featurize_docs(const char* const* docs, const int64_t* lens, int64_t count,
                                       const int64_t* batch_override, int32_t threads) {
  auto* b = new (std::nothrow) dippm_feat_batch;
  if (!b) return nullptr;
  b->res.resize(count > 0 ? (size_t)count : 0);
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<int64_t>(nt, std::max<int64_t>(count, 1));
  // dynamic scheduling in small grains: document sizes are heavy-tailed (power-law node
  // counts) and the host may be shared with other work, so static slices straggle
  std::atomic<int64_t> next{0};
  const int64_t grain = 4;
  auto work = [&] {
    for (int64_t i0; (i0 = next.fetch_add(grain, std::memory_order_relaxed)) < count;)
      for (int64_t i = i0; i < std::min(count, i0 + grain); ++i)
        featurize_one(docs[i], lens[i], batch_override ? batch_override[i] : 0, b->res[i]);
  };
  if (nt <= 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();  // the calling thread is one of the workers
    for (auto& th : pool) th.join();
  }
  return b;
}

int64_t dippm_feat_count(const dippm_feat_batch* b) { return b ? (int64_t)b->res.size() : 0; }

int32_t dippm_feat_status(const dippm_feat_batch* b, int64_t i, char* msg, int64_t cap) {
  const Result& r = b->res[i];
  if (msg && cap > 0) {
    const size_t n = std::min<size_t>(r.msg.size(), (size_t)cap - 1);
    memcpy(msg, r.msg.data(), n);
    msg[n] = 0;
  }
  return r.status;
}

int64_t dippm_feat_name(const dippm_feat_batch* b, int64_t i, char* buf, int64_t cap) {
  const std::string& s = b->res[i].name;
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(s.size(), (size_t)cap - 1);
    memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return (int64_t)s.size();
}

void dippm_feat_sizes(const dippm_feat_batch* b, int64_t* num_nodes, int64_t* num_edges, int64_t* total_nodes,
                      int64_t* total_edges) {
  int64_t tn = 0, te = 0;
  for (size_t i = 0; i < b->res.size(); ++i) {
    const Result& r = b->res[i];
    if (num_nodes) num_nodes[i] = r.n;
    if (num_edges) num_edges[i] = (int64_t)r.edges.size();
    tn += r.n;
    te += (int64_t)r.edges.size();
  }
  if (total_nodes) *total_nodes = tn;
  if (total_edges) *total_edges = te;
}

}  // extern "C"

namespace {
// node / edge offsets of every document, and a parallel loop over document ranges whose
// output slices are disjoint
void doc_offsets(const dippm_feat_batch* b, std::vector<int64_t>& no, std::vector<int64_t>& eo) {
  const size_t G = b->res.size();
  no.assign(G + 1, 0);
  eo.assign(G + 1, 0);
  for (size_t i = 0; i < G; ++i) {
    no[i + 1] = no[i] + b->res[i].n;
    eo[i + 1] = eo[i] + (int64_t)b->res[i].edges.size();
  }
}
template <class F>
void parallel_docs(size_t G, F&& work) {  // work(i0, i1) over dynamically claimed document ranges
  const int nt = (int)std::min<size_t>(std::max(1u, std::thread::hardware_concurrency()), std::max<size_t>(G / 64, 1));
  if (nt <= 1) {
    work((size_t)0, G);
    return;
  }
  std::atomic<size_t> next{0};
  const size_t grain = 16;
  auto loop = [&] {
    for (size_t i0; (i0 = next.fetch_add(grain, std::memory_order_relaxed)) < G;) work(i0, std::min(G, i0 + grain));
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(loop);
  loop();
  for (auto& th : pool) th.join();
}
}  // namespace

extern "C" {

void dippm_feat_export(const dippm_feat_batch* b, double* x, int64_t* edges, int64_t* fs_int, float* x32) {
  std::vector<int64_t> no, eo;
  doc_offsets(b, no, eo);
  parallel_docs(b->res.size(), [&](size_t i0, size_t i1) {
    for (size_t i = i0; i < i1; ++i) {
      const Result& r = b->res[i];
      if (x && r.n) memcpy(x + no[i] * 32, r.x.data(), sizeof(double) * 32 * (size_t)r.n);
      if (x32)
        for (int64_t k = 0; k < r.n * 32; ++k) x32[no[i] * 32 + k] = (float)r.x[(size_t)k];
      if (edges)
        for (size_t k = 0; k < r.edges.size(); ++k) {
          edges[2 * (eo[i] + (int64_t)k)] = r.edges[k].first;
          edges[2 * (eo[i] + (int64_t)k) + 1] = r.edges[k].second;
        }
      if (fs_int)
        for (int k = 0; k < 5; ++k) fs_int[i * 5 + k] = r.fs[k];
    }
  });
}

void dippm_feat_collate(const dippm_feat_batch* b, float* x32, int64_t* src, int64_t* dst, int32_t* graph_ptr,
                        int64_t* edge_ptr, double* fs64) {
  std::vector<int64_t> no, eo;
  doc_offsets(b, no, eo);
  const size_t G = b->res.size();
  if (graph_ptr)
    for (size_t i = 0; i <= G; ++i) graph_ptr[i] = (int32_t)no[i];
  if (edge_ptr)
    for (size_t i = 0; i <= G; ++i) edge_ptr[i] = eo[i];
  parallel_docs(G, [&](size_t i0, size_t i1) {
    for (size_t i = i0; i < i1; ++i) {
      const Result& r = b->res[i];
      if (x32)
        for (int64_t k = 0; k < r.n * 32; ++k) x32[no[i] * 32 + k] = (float)r.x[(size_t)k];
      for (size_t k = 0; k < r.edges.size(); ++k) {
        if (src) src[eo[i] + (int64_t)k] = no[i] + r.edges[k].first;
        if (dst) dst[eo[i] + (int64_t)k] = no[i] + r.edges[k].second;
      }
      if (fs64)
        for (int k = 0; k < 5; ++k) fs64[i * 5 + k] = std::log1p((double)r.fs[k]);
    }
  });
}

int64_t dippm_feat_meta(const dippm_feat_batch* b, int32_t* status, double* fs_log, int64_t* name_off, char* names,
                        int64_t names_cap) {
  int64_t off = 0;
  for (size_t i = 0; i < b->res.size(); ++i) {
    const Result& r = b->res[i];
    if (status) status[i] = r.status;
    if (fs_log)
      for (int k = 0; k < 5; ++k) fs_log[i * 5 + k] = std::log1p((double)r.fs[k]);  // math.log1p(int) semantics
    if (name_off) name_off[i] = off;
    if (names && off + (int64_t)r.name.size() <= names_cap) memcpy(names + off, r.name.data(), r.name.size());
    off += (int64_t)r.name.size();
  }
  if (name_off) name_off[b->res.size()] = off;
  return off;
}

void dippm_feat_free(dippm_feat_batch* b) { delete b; }

}  // extern "C"
