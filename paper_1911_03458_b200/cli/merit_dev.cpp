// merit-dev — the reference CLI's `run` path on the B200.
//
//   merit-dev run --manifest M.json [--tile 16x8,5x5] [--out out.mrt] [--dry-run]
//   merit-dev info
//
// Reads the reference's workload manifest (tools/merit.cpp:102-118: view_a,
// view_b, program, tensor_a, tensor_b, optional tiling; views / programs in
// the serialize.hpp:104-184 layout) and MRT1 tensors (tensor.hpp:123-163),
// runs the workload through the C ABI (include/merit_dev.h) and prints the
// reference's `run` report as JSON (tools/merit.cpp:139-175: p_shape,
// a_shape, traffic + naive_unrolled_words with --tile, output_shape,
// checksum) plus a "device" object (kernel, plan).  --out writes the output
// as MRT1.  --dry-run lowers and reports the plan without a GPU.  Exit codes
// follow the reference CLI: 2 for usage errors, 1 for other errors.
//
// Host code only: the JSON reader is a small recursive-descent parser for
// the manifest schema (nlohmann/json, the reference's dependency, is not a
// dependency here).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "merit_dev.h"

namespace {

// ------------------------------------------------------------ errors ----
struct CliError : std::runtime_error {
  merit_status code;
  CliError(merit_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(merit_status c, const std::string& m) { throw CliError(c, m); }

// -------------------------------------------------------------- JSON ----
struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  const Json* find(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Json& at(const std::string& k) const {
    const Json* v = kind == Obj ? find(k) : nullptr;
    if (!v) fail(MERIT_E_BAD_PARAMS, "manifest: missing key \"" + k + "\"");
    return *v;
  }
  int64_t as_int() const {
    if (kind != Num || std::floor(num) != num) fail(MERIT_E_BAD_PARAMS, "manifest: expected an integer");
    return static_cast<int64_t>(num);
  }
  double as_num() const {
    if (kind != Num) fail(MERIT_E_BAD_PARAMS, "manifest: expected a number");
    return num;
  }
  const std::string& as_str() const {
    if (kind != Str) fail(MERIT_E_BAD_PARAMS, "manifest: expected a string");
    return str;
  }
  const std::vector<Json>& as_arr() const {
    if (kind != Arr) fail(MERIT_E_BAD_PARAMS, "manifest: expected an array");
    return arr;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Json parse() {
    Json v = value();
    ws();
    if (i_ != s_.size()) err("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
  [[noreturn]] void err(const std::string& m) {
    fail(MERIT_E_BAD_PARAMS, "manifest JSON: " + m + " at offset " + std::to_string(i_));
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t')) ++i_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (s_.compare(i_, n, w) == 0) { i_ += n; return true; }
    return false;
  }
  Json value() {
    ws();
    if (i_ >= s_.size()) err("unexpected end");
    const char c = s_[i_];
    Json v;
    if (c == '{') {
      v.kind = Json::Obj;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
      for (;;) {
        ws();
        Json k = value();
        if (k.kind != Json::Str) err("object key must be a string");
        ws();
        if (i_ >= s_.size() || s_[i_] != ':') err("expected ':'");
        ++i_;
        v.obj.emplace_back(k.str, value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
        if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
        err("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Json::Arr;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
        if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
        err("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Json::Str;
      ++i_;
      while (i_ < s_.size() && s_[i_] != '"') {
        if (s_[i_] == '\\') {
          ++i_;
          if (i_ >= s_.size()) err("bad escape");
          const char e = s_[i_];
          v.str.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e);
        } else {
          v.str.push_back(s_[i_]);
        }
        ++i_;
      }
      if (i_ >= s_.size()) err("unterminated string");
      ++i_;
      return v;
    }
    if (lit("true")) { v.kind = Json::Bool; v.b = true; return v; }
    if (lit("false")) { v.kind = Json::Bool; return v; }
    if (lit("null")) return v;
    char* end = nullptr;
    v.num = std::strtod(s_.c_str() + i_, &end);
    if (end == s_.c_str() + i_) err("unexpected character");
    v.kind = Json::Num;
    i_ = static_cast<size_t>(end - s_.c_str());
    return v;
  }
};

std::string read_file(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) fail(MERIT_E_USAGE, "cannot open " + path);
  std::stringstream ss;
  ss << is.rdbuf();
  return ss.str();
}

// -------------------------------------------------------------- MRT1 ----
struct Tensor {
  int dtype = 0;  // 0 REAL32, 1 FIX16
  int frac_bits = 0;
  std::vector<int64_t> shape;
  std::vector<uint8_t> payload;  // little-endian words
  int64_t size() const {
    int64_t n = 1;
    for (int64_t e : shape) n *= e;
    return n;
  }
};

Tensor read_mrt1(const std::string& path) {  // tensor.hpp:141-163
  const std::string d = read_file(path);
  size_t pos = 0;
  auto need = [&](size_t n) {
    if (pos + n > d.size()) fail(MERIT_E_TRUNCATED_PAYLOAD, "unexpected EOF");
  };
  auto u8 = [&]() { need(1); return static_cast<uint32_t>(static_cast<uint8_t>(d[pos++])); };
  auto u16 = [&]() { const uint32_t lo = u8(); return lo | (u8() << 8); };
  auto u32 = [&]() { const uint32_t lo = u16(); return lo | (u16() << 16); };
  if (d.size() < 4 || std::memcmp(d.data(), "MRT1", 4) != 0) fail(MERIT_E_BAD_MAGIC, "bad magic, expected MRT1");
  pos = 4;
  Tensor t;
  t.dtype = static_cast<int>(u8());
  t.frac_bits = static_cast<int>(u8());
  if (t.dtype > 1) fail(MERIT_E_UNKNOWN_DTYPE, "unknown dtype code");
  const uint32_t rank = u16();
  for (uint32_t i = 0; i < rank; ++i) t.shape.push_back(u32());
  if (rank < 1) fail(MERIT_E_TRUNCATED_PAYLOAD, "rank must be >= 1");
  for (int64_t e : t.shape)
    if (e < 1) fail(MERIT_E_BAD_PARAMS, "extents must be >= 1");
  if (t.dtype == 0) t.frac_bits = 0;
  const size_t bytes = static_cast<size_t>(t.size()) * (t.dtype == 0 ? 4 : 2);
  need(bytes);
  t.payload.assign(d.begin() + pos, d.begin() + pos + bytes);
  return t;
}

void write_mrt1(const std::string& path, int dtype, int frac_bits, const std::vector<int64_t>& shape,
                const void* data, size_t bytes) {  // tensor.hpp:123-139
  std::ofstream os(path, std::ios::binary);
  if (!os) fail(MERIT_E_USAGE, "cannot write " + path);
  auto u8 = [&](uint32_t v) { os.put(static_cast<char>(v & 0xff)); };
  auto u16 = [&](uint32_t v) { u8(v); u8(v >> 8); };
  auto u32 = [&](uint32_t v) { u16(v & 0xffff); u16(v >> 16); };
  os.write("MRT1", 4);
  u8(static_cast<uint32_t>(dtype));
  u8(static_cast<uint32_t>(frac_bits));
  u16(static_cast<uint32_t>(shape.size()));
  for (int64_t e : shape) u32(static_cast<uint32_t>(e));
  os.write(static_cast<const char*>(data), static_cast<std::streamsize>(bytes));  // x86: little-endian
}

// ----------------------------------------------------- manifest -> ABI ---
void fill_view(merit_view_spec& v, const Json& j) {  // serialize.hpp:119-131
  v = merit_view_spec{};
  auto shape = [&](const char* key, int64_t* dst, int32_t& rank) {
    const auto& a = j.at(key).as_arr();
    if (a.size() > MERIT_MAX_RANK) fail(MERIT_E_BAD_PARAMS, std::string("manifest: ") + key + " rank too large");
    rank = static_cast<int32_t>(a.size());
    for (size_t i = 0; i < a.size(); ++i) dst[i] = a[i].as_int();
  };
  shape("source_shape", v.src_shape, v.src_rank);
  shape("p_shape", v.p_shape, v.p_rank);
  shape("a_shape", v.a_shape, v.a_rank);
  const auto& terms = j.at("terms").as_arr();
  if (terms.size() > MERIT_MAX_TERMS) fail(MERIT_E_BAD_PARAMS, "manifest: too many terms");
  v.n_terms = static_cast<int32_t>(terms.size());
  for (size_t t = 0; t < terms.size(); ++t)
    v.terms[t] = merit_view_term{static_cast<int32_t>(terms[t].at("component").as_int()),
                                 static_cast<int32_t>(terms[t].at("axis").as_int()),
                                 terms[t].at("stride").as_int(), terms[t].at("offset").as_int()};
  v.boundary = MERIT_ZERO_PAD;
  if (const Json* b = j.find("boundary")) {
    const std::string& s = b->as_str();
    if (s == "ZERO_PAD") v.boundary = MERIT_ZERO_PAD;
    else if (s == "CLAMP") v.boundary = MERIT_CLAMP;
    else if (s == "REJECT") v.boundary = MERIT_REJECT;
    else fail(MERIT_E_BAD_PARAMS, "unknown boundary " + s);
  }
}

void operand(const std::string& s, int32_t& kind, int32_t& reg) {  // serialize.hpp:57-70
  reg = 0;
  if (s == "a") { kind = 1; return; }
  if (s == "b") { kind = 2; return; }
  if (s == "_") { kind = 3; return; }
  if (s.size() >= 2 && s[0] == 'r') {
    const int id = std::atoi(s.c_str() + 1);
    if (id < 0 || id > 15 || s.find_first_not_of("0123456789", 1) != std::string::npos)
      fail(MERIT_E_BAD_PARAMS, "register id out of range: " + s);
    kind = 0;
    reg = id;
    return;
  }
  fail(MERIT_E_BAD_PARAMS, "bad operand " + s);
}

struct Program {  // owns the arrays merit_program points into
  std::vector<int32_t> seg_len;
  std::vector<merit_alu_instr> instrs;
  std::vector<double> constants;
  std::vector<std::vector<double>> samples;
  std::vector<merit_lookup_table> tables;
};

void fill_program(merit_program& pc, Program& P, const Json& j) {  // serialize.hpp:160-184
  static const char* names[] = {"ADD", "SUB", "L1", "MAC", "MAX", "MIN", "SEL", "BAND",
                                "BOR", "BXOR", "BNOT", "IDX", "LUT", "MOVC", "DIV"};
  for (const Json& seg : j.at("segments").as_arr()) {
    P.seg_len.push_back(static_cast<int32_t>(seg.as_arr().size()));
    for (const Json& in : seg.as_arr()) {
      merit_alu_instr c{};
      const std::string& op = in.at("op").as_str();
      c.op = -1;
      for (int k = 0; k < 15; ++k)
        if (op == names[k]) c.op = k;
      if (c.op < 0) fail(MERIT_E_BAD_PARAMS, "unknown op " + op);
      const std::string& dst = in.at("dst").as_str();
      if (dst == "out") {
        c.dst_out = 1;
      } else {
        int32_t kind;
        operand(dst, kind, c.dst_reg);
        if (kind != 0) fail(MERIT_E_BAD_PARAMS, "bad destination " + dst);
      }
      operand(in.at("a").as_str(), c.a_kind, c.a_reg);
      operand(in.at("b").as_str(), c.b_kind, c.b_reg);
      operand(in.at("c").as_str(), c.c_kind, c.c_reg);
      if (const Json* v = in.find("shift")) c.shift = static_cast<int32_t>(v->as_int());
      if (const Json* v = in.find("aux")) c.aux = static_cast<int32_t>(v->as_int());
      P.instrs.push_back(c);
    }
  }
  if (const Json* cs = j.find("constants"))
    for (const Json& c : cs->as_arr()) P.constants.push_back(c.as_num());
  if (const Json* ts = j.find("tables")) {
    P.samples.reserve(ts->as_arr().size());
    for (const Json& t : ts->as_arr()) {
      P.samples.emplace_back();
      for (const Json& s : t.at("samples").as_arr()) P.samples.back().push_back(s.as_num());
      const Json* cl = t.find("clamp");
      P.tables.push_back(merit_lookup_table{t.at("lo").as_num(), t.at("hi").as_num(),
                                            static_cast<int32_t>(P.samples.back().size()),
                                            (cl && cl->kind == Json::Bool && !cl->b) ? 0 : 1,
                                            P.samples.back().data()});
    }
  }
  pc = merit_program{};
  pc.depth = static_cast<int32_t>(j.at("depth").as_int());
  pc.outputs = 1;
  if (const Json* o = j.find("outputs")) pc.outputs = static_cast<int32_t>(o->as_int());
  pc.n_segments = static_cast<int32_t>(P.seg_len.size());
  pc.n_constants = static_cast<int32_t>(P.constants.size());
  pc.n_tables = static_cast<int32_t>(P.tables.size());
  pc.seg_len = P.seg_len.data();
  pc.instrs = P.instrs.data();
  pc.constants = P.constants.data();
  pc.tables = P.tables.data();
}

std::vector<int64_t> int_list(const std::string& s, char sep) {  // tools/merit.cpp:25-35
  std::vector<int64_t> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, sep)) {
    if (item.empty()) fail(MERIT_E_USAGE, "empty list item");
    out.push_back(std::stoll(item));
  }
  if (out.empty()) fail(MERIT_E_USAGE, "empty list");
  return out;
}

std::string json_list(const std::vector<int64_t>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + std::to_string(v[i]);
  return s + "]";
}

std::string json_str(const std::string& v) {
  std::string s = "\"";
  for (char c : v) {
    if (c == '"' || c == '\\') s.push_back('\\');
    s.push_back(c);
  }
  return s + "\"";
}

void check(merit_status st) {
  if (st != MERIT_OK) fail(st, merit_dev_last_error());
}

int cmd_run(const std::string& manifest, std::string tile, const std::string& out_path, bool dry_run) {
  if (manifest.empty()) fail(MERIT_E_USAGE, "run needs --manifest (templates: python -m paper_1911_03458_b200.manifest)");
  const Json j = Parser(read_file(manifest)).parse();
  const std::string dir = manifest.find('/') == std::string::npos ? "" : manifest.substr(0, manifest.rfind('/') + 1);
  auto path_of = [&](const std::string& p) { return (!p.empty() && p[0] == '/') ? p : dir + p; };
  if (tile.empty())
    if (const Json* t = j.find("tiling")) tile = t->as_str();

  merit_workload_desc d{};
  fill_view(d.view_a, j.at("view_a"));
  fill_view(d.view_b, j.at("view_b"));
  Program P;
  fill_program(d.program, P, j.at("program"));
  const Tensor ta = read_mrt1(path_of(j.at("tensor_a").as_str()));
  const Tensor tb = read_mrt1(path_of(j.at("tensor_b").as_str()));
  d.dtype_a = ta.dtype ? MERIT_I16 : MERIT_F32;
  d.dtype_b = tb.dtype ? MERIT_I16 : MERIT_F32;
  d.dtype_out = d.dtype_a;
  d.frac_bits = ta.frac_bits;
  // Workload::validate's source-shape check (engine.hpp:35-36)
  auto same = [](const Tensor& t, const merit_view_spec& v) {
    if (static_cast<int>(t.shape.size()) != v.src_rank) return false;
    for (int i = 0; i < v.src_rank; ++i)
      if (t.shape[i] != v.src_shape[i]) return false;
    return true;
  };
  if (!same(ta, d.view_a) || !same(tb, d.view_b)) fail(MERIT_E_BAD_PARAMS, "source shape mismatch");

  struct PlanGuard {
    merit_plan* p = nullptr;
    ~PlanGuard() { merit_dev_plan_destroy(p); }
  } plan;
  check(merit_dev_plan_create(&d, &plan.p));
  merit_plan_info info{};
  check(merit_dev_plan_query(plan.p, &info));

  std::vector<int64_t> p_shape(d.view_a.p_shape, d.view_a.p_shape + d.view_a.p_rank);
  std::vector<int64_t> a_shape(d.view_a.a_shape, d.view_a.a_shape + d.view_a.a_rank);
  std::vector<int64_t> out_shape(info.out_shape, info.out_shape + info.out_rank);
  std::ostringstream rep;
  rep << "{\n  \"template\": \"(manifest)\",\n  \"seed\": 0,\n  \"p_shape\": " << json_list(p_shape)
      << ",\n  \"a_shape\": " << json_list(a_shape);
  if (!tile.empty()) {  // "16x8,5x5" (tools/merit.cpp:37-44)
    const auto comma = tile.find(',');
    if (comma == std::string::npos) fail(MERIT_E_USAGE, "tile must be PxP...,AxA...");
    const auto tp = int_list(tile.substr(0, comma), 'x');
    const auto tt = int_list(tile.substr(comma + 1), 'x');
    if (static_cast<int>(tp.size()) != d.view_a.p_rank || static_cast<int>(tt.size()) != d.view_a.a_rank)
      fail(MERIT_E_BAD_PARAMS, "tile rank mismatch");
    merit_traffic_report r{};
    check(merit_dev_tiled_traffic(plan.p, tp.data(), tt.data(), &r));
    int64_t naive = 1;
    for (int64_t e : p_shape) naive *= e;
    for (int64_t e : a_shape) naive *= e;
    rep << ",\n  \"traffic\": {\"dram_read_words_a\": " << r.dram_read_words_a
        << ", \"dram_read_words_b\": " << r.dram_read_words_b << ", \"dram_write_words\": " << r.dram_write_words
        << ", \"scratchpad_peak_words_a\": " << r.scratchpad_peak_words_a
        << ", \"scratchpad_peak_words_b\": " << r.scratchpad_peak_words_b << ", \"passes\": " << r.passes
        << ", \"macs\": " << r.macs << "},\n  \"naive_unrolled_words\": " << naive;
  }
  rep << ",\n  \"output_shape\": " << json_list(out_shape);
  if (!dry_run) {
    const size_t elem = d.dtype_out == MERIT_I16 ? 2 : 4;
    std::vector<uint8_t> out(static_cast<size_t>(info.out_elems) * elem);
    check(merit_dev_run_host(plan.p, ta.payload.data(), tb.payload.data(), out.data(), nullptr, nullptr));
    double checksum = 0;  // tools/merit.cpp:72-79
    for (int64_t i = 0; i < info.out_elems; ++i) {
      if (elem == 4) {
        float v;
        std::memcpy(&v, out.data() + 4 * i, 4);
        checksum += v;
      } else {
        int16_t v;
        std::memcpy(&v, out.data() + 2 * i, 2);
        checksum += v;
      }
    }
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.17g", checksum);
    rep << ",\n  \"checksum\": " << buf;
    if (!out_path.empty())
      write_mrt1(out_path, elem == 2 ? 1 : 0, elem == 2 ? ta.frac_bits : 0, out_shape, out.data(), out.size());
  }
  rep << ",\n  \"device\": {\"kernel\": " << json_str(dry_run ? "" : merit_dev_last_kernel())
      << ", \"plan\": " << json_str(info.description) << ", \"dry_run\": " << (dry_run ? "true" : "false")
      << "}\n}\n";
  std::cout << rep.str();
  return 0;
}

const char* kUsage =
    "usage: merit-dev run --manifest M.json [--tile PxP..,AxA..] [--out out.mrt] [--dry-run]\n"
    "       merit-dev info\n";

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage;
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "info") {
      std::cout << "{\"build\": " << json_str(merit_dev_build_info()) << ", \"abi\": " << merit_dev_abi_version()
                << "}\n";
      return 0;
    }
    if (cmd != "run") fail(MERIT_E_USAGE, "unknown subcommand " + cmd);
    std::string manifest, tile, out;
    bool dry = false;
    for (int i = 2; i < argc; ++i) {
      const std::string a = argv[i];
      auto next = [&]() -> std::string {
        if (i + 1 >= argc) fail(MERIT_E_USAGE, a + " needs a value");
        return argv[++i];
      };
      if (a == "--manifest") manifest = next();
      else if (a == "--tile") tile = next();
      else if (a == "--out") out = next();
      else if (a == "--dry-run") dry = true;
      else if (a == "--json") {}  // output is always JSON (tools/merit.cpp:328)
      else fail(MERIT_E_USAGE, "unknown option " + a);
    }
    return cmd_run(manifest, tile, out, dry);
  } catch (const CliError& e) {
    std::cerr << "error: " << e.what() << "\n";
    if (e.code == MERIT_E_USAGE) std::cerr << kUsage;
    return e.code == MERIT_E_USAGE ? 2 : 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
