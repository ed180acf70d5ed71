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
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <string>
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
struct J {
  enum T { NUL, BOOL, INT, FLT, STR, ARR, OBJ } t = NUL;
  bool b = false;
  int64_t i = 0;
  double f = 0.0;
  std::string s;
  std::vector<J> a;
  std::vector<std::pair<std::string, J>> o;

  const J* get(const char* key) const {  // last duplicate wins (Python dict semantics)
    const J* r = nullptr;
    for (const auto& kv : o)
      if (kv.first == key) r = &kv.second;
    return r;
  }
  bool is_int() const { return t == INT; }                 // isinstance(v, int) and not bool
  bool is_num() const { return t == INT || t == FLT; }     // (int, float), not bool
  double num() const { return t == INT ? (double)i : f; }  // float(v)
};

struct Parser {
  const char* p;
  const char* e;
  int depth = 0;
  [[noreturn]] void bad(const char* what) {
    fail(DIPPM_FEAT_MALFORMED_DOCUMENT, std::string("invalid JSON: ") + what);
  }
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool lit(const char* w) {
    size_t n = strlen(w);
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
      char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= (uint32_t)(c - '0');
      else if (c >= 'a' && c <= 'f') v |= (uint32_t)(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= (uint32_t)(c - 'A' + 10);
      else bad("bad \\u escape");
    }
    return v;
  }
  std::string str() {
    ++p;  // opening quote
    std::string out;
    while (true) {
      if (p >= e) bad("unterminated string");
      unsigned char c = (unsigned char)*p++;
      if (c == '"') break;
      if (c < 0x20) bad("control character in string");
      if (c != '\\') {
        out += (char)c;
        continue;
      }
      if (p >= e) bad("unterminated escape");
      char x = *p++;
      switch (x) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00 && e - p >= 6 && p[0] == '\\' && p[1] == 'u') {
            const char* save = p;
            p += 2;
            uint32_t lo = hex4();
            if (lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            else p = save;
          }
          put_utf8(out, cp);
          break;
        }
        default: bad("bad escape");
      }
    }
    return out;
  }
  J number() {
    const char* s0 = p;
    if (p < e && *p == '-') ++p;
    if (p < e && *p == 'I') {  // -Infinity
      if (!lit("Infinity")) bad("bad literal");
      J v;
      v.t = J::FLT;
      v.f = -INFINITY;
      return v;
    }
    if (p >= e || !(*p >= '0' && *p <= '9')) bad("bad number");
    if (*p == '0') ++p;
    else while (p < e && *p >= '0' && *p <= '9') ++p;
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
    std::string tok(s0, p - s0);
    J v;
    if (flt) {
      v.t = J::FLT;
      v.f = strtod(tok.c_str(), nullptr);  // correctly rounded, like Python's float()
    } else {
      errno = 0;
      char* end = nullptr;
      long long x = strtoll(tok.c_str(), &end, 10);
      if (errno == ERANGE) fail(DIPPM_FEAT_UNSUPPORTED, "integer " + tok + " does not fit in 64 bits");
      v.t = J::INT;
      v.i = (int64_t)x;
    }
    return v;
  }
  J value() {
    if (++depth > 512) bad("nesting too deep");
    ws();
    if (p >= e) bad("unexpected end");
    J v;
    char c = *p;
    if (c == '{') {
      ++p;
      v.t = J::OBJ;
      ws();
      if (p < e && *p == '}') {
        ++p;
      } else {
        while (true) {
          ws();
          if (p >= e || *p != '"') bad("expected key");
          std::string k = str();
          ws();
          if (p >= e || *p != ':') bad("expected ':'");
          ++p;
          J val = value();
          v.o.emplace_back(std::move(k), std::move(val));
          ws();
          if (p < e && *p == ',') { ++p; continue; }
          if (p < e && *p == '}') { ++p; break; }
          bad("expected ',' or '}'");
        }
      }
    } else if (c == '[') {
      ++p;
      v.t = J::ARR;
      ws();
      if (p < e && *p == ']') {
        ++p;
      } else {
        while (true) {
          v.a.push_back(value());
          ws();
          if (p < e && *p == ',') { ++p; continue; }
          if (p < e && *p == ']') { ++p; break; }
          bad("expected ',' or ']'");
        }
      }
    } else if (c == '"') {
      v.t = J::STR;
      v.s = str();
    } else if (lit("true")) {
      v.t = J::BOOL;
      v.b = true;
    } else if (lit("false")) {
      v.t = J::BOOL;
    } else if (lit("null")) {
      v.t = J::NUL;
    } else if (lit("NaN")) {
      v.t = J::FLT;
      v.f = NAN;
    } else if (lit("Infinity")) {
      v.t = J::FLT;
      v.f = INFINITY;
    } else {
      v = number();
    }
    --depth;
    return v;
  }
};

J parse_json(const char* s, int64_t n) {
  Parser P{s, s + n};
  J v = P.value();
  P.ws();
  if (P.p != P.e) P.bad("extra data");
  return v;
}

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

// parse_graph_json graph_ir.py:212-297
Graph parse_graph(const char* text, int64_t len) {
  J doc = parse_json(text, len);
  if (doc.t != J::OBJ) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "top-level value must be an object");
  const J* raw_nodes = doc.get("nodes");
  if (!raw_nodes || raw_nodes->t != J::ARR || raw_nodes->a.empty())
    fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "\"nodes\" must be a non-empty list");
  const J* outputs = doc.get("outputs");
  bool ok = outputs && outputs->t == J::ARR && !outputs->a.empty();
  if (ok)
    for (const J& o : outputs->a)
      if (!(o.t == J::INT || o.t == J::BOOL)) ok = false;  // isinstance(o, int): bool is an int
  if (!ok) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "\"outputs\" must be a non-empty list of node ids");
  const J* batch = doc.get("batch");
  if (!batch || batch->t != J::INT || batch->i < 1)
    fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "\"batch\" must be a positive integer");
  const J* name = doc.get("name");
  if (name && name->t != J::STR) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "\"name\" must be a string");

  std::unordered_map<int64_t, size_t> by_id;  // id -> entry index (document order kept in `order_doc`)
  std::vector<int64_t> order_doc;
  std::vector<Node> entries;
  for (const J& ent : raw_nodes->a) {
    if (ent.t != J::OBJ) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "every node must be an object");
    const J* idj = ent.get("id");
    if (!idj || idj->t != J::INT || idj->i < 0)
      fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "node id must be a non-negative integer");
    const int64_t nid = idj->i;
    if (by_id.count(nid)) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "duplicate node id " + I(nid));
    const J* op = ent.get("op");
    if (!op || op->t != J::STR || op->s.empty())
      fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "node " + I(nid) + ": missing operator name");
    Node n;
    n.raw = op->s;
    const J* ins = ent.get("inputs");
    if (ins) {
      bool good = ins->t == J::ARR;
      if (good)
        for (const J& x : ins->a)
          if (x.t != J::INT) good = false;
      if (!good) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "node " + I(nid) + ": inputs must be a list of node ids");
      for (const J& x : ins->a) n.inputs.push_back(x.i);
    }
    const J* attrs = ent.get("attrs");
    if (attrs) {
      bool good = attrs->t == J::OBJ;
      if (good)
        for (const auto& kv : attrs->o)
          if (!kv.second.is_num()) good = false;
      if (!good) fail(DIPPM_FEAT_MALFORMED_DOCUMENT, "node " + I(nid) + ": attrs must map names to numbers");
      for (const auto& kv : attrs->o)
        for (int a = 0; a < 12; ++a)
          if (kv.first == kAttrs[a]) {  // later duplicates overwrite (dict semantics)
            n.has_attr[a] = true;
            n.attr[a] = kv.second.num();
            n.attr_int[a] = kv.second.t == J::INT;
            n.attr_i[a] = kv.second.i;
          }
    }
    const J* shp = ent.get("out_shape");
    if (shp && shp->t != J::NUL) {
      if (shp->t != J::ARR) fail(DIPPM_FEAT_BAD_SHAPE, "node " + I(nid) + ": out_shape must be a list");
      if (shp->a.size() < 1 || shp->a.size() > 4)
        fail(DIPPM_FEAT_BAD_SHAPE, "node " + I(nid) + ": shape rank " + I((int64_t)shp->a.size()) + " outside [1, 4]");
      for (const J& d : shp->a) {
        if (d.t != J::INT || d.i < 1)
          fail(DIPPM_FEAT_BAD_SHAPE, "node " + I(nid) + ": shape entry is not a positive integer");
        n.shape.push_back(d.i);
      }
      n.has_shape = true;
    }
    by_id[nid] = entries.size();
    order_doc.push_back(nid);
    entries.push_back(std::move(n));
  }
  for (size_t k = 0; k < entries.size(); ++k)
    for (int64_t src : entries[k].inputs)
      if (!by_id.count(src))
        fail(DIPPM_FEAT_DANGLING_REFERENCE, "node " + I(order_doc[k]) + " references missing input " + I(src));
  for (const J& o : outputs->a) {
    const int64_t oid = o.t == J::BOOL ? (int64_t)o.b : o.i;
    if (!by_id.count(oid)) fail(DIPPM_FEAT_DANGLING_REFERENCE, "output id " + I(oid) + " does not exist");
  }
  // _topological_order: Kahn over a min-heap of original ids, inputs counted with multiplicity
  std::unordered_map<int64_t, std::vector<int64_t>> consumers;
  std::unordered_map<int64_t, int64_t> pending;
  for (size_t k = 0; k < entries.size(); ++k) {
    pending[order_doc[k]] = (int64_t)entries[k].inputs.size();
    for (int64_t src : entries[k].inputs) consumers[src].push_back(order_doc[k]);
  }
  std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> heap;
  for (int64_t nid : order_doc)
    if (pending[nid] == 0) heap.push(nid);
  std::vector<int64_t> order;
  while (!heap.empty()) {
    const int64_t nid = heap.top();
    heap.pop();
    order.push_back(nid);
    auto it = consumers.find(nid);
    if (it != consumers.end())
      for (int64_t c : it->second)
        if (--pending[c] == 0) heap.push(c);
  }
  if (order.size() != entries.size()) {
    std::vector<int64_t> stuck;
    std::unordered_set<int64_t> done(order.begin(), order.end());
    for (int64_t nid : order_doc)
      if (!done.count(nid)) stuck.push_back(nid);
    std::sort(stuck.begin(), stuck.end());
    fail(DIPPM_FEAT_CYCLIC_GRAPH, "nodes " + shape_str(stuck) + " form a dependency cycle");
  }
  std::unordered_map<int64_t, int64_t> remap;
  for (size_t k = 0; k < order.size(); ++k) remap[order[k]] = (int64_t)k;
  Graph g;
  g.batch = batch->i;
  g.name = name ? name->s : "";
  g.nodes.reserve(order.size());
  for (int64_t old : order) {
    Node n = entries[by_id[old]];
    for (auto& i : n.inputs) i = remap[i];
    const std::string tail = op_tail(n.raw);
    n.kind = OTHER;
    for (int k = 0; k < 16; ++k)
      if (tail == kKinds[k]) n.kind = k;
    n.is_op = true;
    for (const char* w : kNonOperator)
      if (tail == w) n.is_op = false;
    g.nodes.push_back(std::move(n));
  }
  for (const J& o : outputs->a) g.outputs.push_back(remap[o.t == J::BOOL ? (int64_t)o.b : o.i]);
  return g;
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
std::vector<int64_t> infer_node(const Node& n, int64_t id, const std::vector<std::vector<int64_t>>& in) {
  const std::string nid = I(id);
  if (n.inputs.empty()) {
    if (!n.has_shape) fail(DIPPM_FEAT_UNDERSPECIFIED, "source node " + nid + " (" + n.raw + ") declares no out_shape");
    return n.shape;
  }
  const int k = n.kind;
  const auto& first = in[0];
  if (k == CONV2D || k == CONV2D_T) {
    if (first.size() != 4)
      fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid + ": " + kKinds[k] + " input must be rank 4, got " + shape_str(first));
    const int64_t kh = attr_int(n, KH), kw = attr_int(n, KW);
    if (kh < 1 || kw < 1) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid + ": " + kKinds[k] + " kernel size missing");
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
      else fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid + ": " + kKinds[k] + " output channels missing");
    }
    const int64_t nn = first[0], h = first[2], w = first[3];
    if (k == CONV2D) return {nn, out_c, conv_spatial(h, kh, sh, ph, dh), conv_spatial(w, kw, sw, pw, dw)};
    return {nn, out_c, (h - 1) * sh - 2 * ph + dh * (kh - 1) + 1, (w - 1) * sw - 2 * pw + dw * (kw - 1) + 1};
  }
  if (k == MAXPOOL || k == AVGPOOL) {
    if (first.size() != 4)
      fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid + ": " + kKinds[k] + " input must be rank 4, got " + shape_str(first));
    const int64_t kh = attr_int(n, KH), kw = attr_int(n, KW);
    if (kh < 1 || kw < 1) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid + ": pool kernel size missing");
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
      fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid + ": global pool input must be rank 4, got " + shape_str(first));
    return {first[0], first[1], 1, 1};
  }
  if (k == DENSE) {
    const int64_t of = attr_int(n, OUTF);
    if (of < 1) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid + ": dense out_features missing");
    std::vector<int64_t> r(first.begin(), first.end() - 1);
    r.push_back(of);
    return r;
  }
  if (k == BMM) {
    if (in.size() != 2) fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid + ": batch_matmul needs exactly 2 inputs");
    const auto &a = in[0], &b = in[1];
    if (a.size() != 3 || b.size() != 3)
      fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid + ": batch_matmul inputs must be rank 3");
    if (a[0] != b[0] || a[2] != b[1]) fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid + ": batch_matmul shapes do not compose");
    return {a[0], a[1], b[2]};
  }
  if (k == ADD || k == MUL) {
    for (size_t j = 1; j < in.size(); ++j)
      if (in[j] != first) fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid + ": elementwise inputs differ");
    return first;
  }
  if (k == CONCAT) {
    if (first.size() < 2) fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid + ": concat inputs must have rank >= 2");
    int64_t ch = 0;
    for (const auto& s : in) {
      bool same = s.size() == first.size() && s[0] == first[0];
      for (size_t d = 2; same && d < s.size(); ++d) same = s[d] == first[d];
      if (!same) fail(DIPPM_FEAT_SHAPE_MISMATCH, "node " + nid + ": concat inputs differ outside channel dim");
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
  std::vector<std::vector<int64_t>> shapes;
  shapes.reserve(g.nodes.size());
  for (size_t k = 0; k < g.nodes.size(); ++k) {
    Node& n = g.nodes[k];
    std::vector<std::vector<int64_t>> in;
    for (int64_t i : n.inputs) in.push_back(shapes[i]);
    std::vector<int64_t> s = infer_node(n, (int64_t)k, in);
    check_shape(s, (int64_t)k);
    shapes.push_back(s);
  }
  for (size_t k = 0; k < g.nodes.size(); ++k) {
    g.nodes[k].shape = shapes[k];
    g.nodes[k].has_shape = true;
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
  std::vector<std::vector<int64_t>> producers(N);
  for (size_t v = 0; v < N; ++v) {
    std::vector<int64_t>& seen = producers[v];
    for (int64_t src : g.nodes[v].inputs) {
      auto add = [&](int64_t c) {
        if (std::find(seen.begin(), seen.end(), c) == seen.end()) seen.push_back(c);
      };
      if (g.nodes[src].is_op) add(src);
      else
        for (int64_t c : producers[src]) add(c);
    }
  }
  std::vector<char> visited(N, 0);
  auto visit = [&](int64_t root) {
    std::vector<std::pair<int64_t, bool>> stack{{root, false}};
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
      const auto& pr = producers[nid];
      for (auto it = pr.rbegin(); it != pr.rend(); ++it)
        if (!visited[*it]) stack.push_back({*it, false});
    }
  };
  for (int64_t out : g.outputs) {
    if (g.nodes[out].is_op) {
      if (!visited[out]) visit(out);
    } else {
      for (int64_t r : producers[out])
        if (!visited[r]) visit(r);
    }
  }
  for (size_t v = 0; v < N; ++v)
    if (g.nodes[v].is_op && !visited[v]) visit((int64_t)v);
  std::vector<int64_t> position(N, -1);
  for (size_t i = 0; i < order.size(); ++i) position[order[i]] = (int64_t)i;
  std::unordered_set<uint64_t> emitted;
  for (int64_t nid : order)
    for (int64_t src : producers[nid]) {
      const uint64_t key = ((uint64_t)position[src] << 32) | (uint64_t)position[nid];
      if (emitted.insert(key).second) edges.push_back({position[src], position[nid]});
    }
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
    const std::string nid = I((int64_t)k);
    if (n.inputs.empty()) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid + ": input shape unavailable");
    const auto& in = g.nodes[n.inputs[0]].shape;
    const auto& out = n.shape;
    if (n.kind == DENSE) {
      __int128 lead = 1;
      for (size_t d = 0; d + 1 < out.size(); ++d) lead *= out[d];
      total += lead * in.back() * out.back();
    } else if (n.kind == BMM) {
      if (out.size() < 3 || in.size() < 3) fail(DIPPM_FEAT_VALUE_ERROR, "node " + nid + ": list index out of range");
      total += (__int128)out[0] * out[1] * out[2] * in[2];
    } else {
      const int64_t kh = attr_int(n, KH), kw = attr_int(n, KW);
      if (kh < 1 || kw < 1) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid + ": kernel size missing");
      int64_t groups = attr_int(n, GROUPS);
      if (!groups) groups = 1;
      if (in.size() != 4 || out.size() != 4) fail(DIPPM_FEAT_UNDERSPECIFIED, "node " + nid + ": conv shapes must be rank 4");
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
    Graph g = parse_graph(doc, len);
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
  auto work = [&](int t) {
    for (int64_t i = t; i < count; i += nt)
      featurize_one(docs[i], lens[i], batch_override ? batch_override[i] : 0, b->res[i]);
  };
  if (nt <= 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work, t);
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

void dippm_feat_export(const dippm_feat_batch* b, double* x, int64_t* edges, int64_t* fs_int, float* x32) {
  int64_t no = 0, eo = 0;
  for (size_t i = 0; i < b->res.size(); ++i) {
    const Result& r = b->res[i];
    if (x && r.n) memcpy(x + no * 32, r.x.data(), sizeof(double) * 32 * (size_t)r.n);
    if (x32)
      for (int64_t k = 0; k < r.n * 32; ++k) x32[no * 32 + k] = (float)r.x[(size_t)k];
    if (edges)
      for (size_t k = 0; k < r.edges.size(); ++k) {
        edges[2 * (eo + (int64_t)k)] = r.edges[k].first;
        edges[2 * (eo + (int64_t)k) + 1] = r.edges[k].second;
      }
    if (fs_int)
      for (int k = 0; k < 5; ++k) fs_int[i * 5 + k] = r.fs[k];
    no += r.n;
    eo += (int64_t)r.edges.size();
  }
}

void dippm_feat_free(dippm_feat_batch* b) { delete b; }

}  // extern "C"
