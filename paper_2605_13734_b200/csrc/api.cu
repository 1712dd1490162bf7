// C ABI (include/kvc.h): plan creation, size queries, encode / decode.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <vector>

#include "kernels.h"
#include "kvc_internal.h"
#include "rc_tables.cuh"

using namespace kvc;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(KVC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- id parser
// Grammar of strategy.py:8-19 (and the same validations: quantize.py:26-62,
// transforms.py:25-30, codecs.py:32-38) plus the extension kinds.
// Python's int() / float() on a str (the reference parses with them,
// strategy.py:68-109): surrounding whitespace, a sign, single underscores
// between digits, any Unicode decimal digit (category Nd, Unicode 15.0 as in
// CPython 3.12), and for float a fraction, an exponent or nan / inf /
// infinity in any case.  Hex and other strtod extensions are rejected as
// Python rejects them.  Ids arrive as UTF-8.
bool utf8_decode(const std::string& s, std::vector<uint32_t>& cps, std::vector<size_t>* starts = nullptr) {
  cps.clear();
  for (size_t i = 0; i < s.size();) {
    const unsigned char c = (unsigned char)s[i];
    int n = c < 0x80 ? 1 : (c >> 5) == 0x6 ? 2 : (c >> 4) == 0xE ? 3 : (c >> 3) == 0x1E ? 4 : 0;
    if (n == 0 || i + n > s.size()) return false;
    uint32_t cp = n == 1 ? c : n == 2 ? (c & 0x1Fu) : n == 3 ? (c & 0x0Fu) : (c & 0x07u);
    for (int k = 1; k < n; ++k) {
      const unsigned char d = (unsigned char)s[i + k];
      if ((d >> 6) != 0x2) return false;
      cp = (cp << 6) | (d & 0x3Fu);
    }
    if (starts) starts->push_back(i);
    cps.push_back(cp);
    i += n;
  }
  if (starts) starts->push_back(s.size());
  return true;
}

// str.isspace(); int() / float() strip the same set minus U+001C..U+001F
bool py_isspace(uint32_t c) {
  return (c >= 0x09 && c <= 0x0D) || (c >= 0x1C && c <= 0x20) || c == 0x85 || c == 0xA0 || c == 0x1680 ||
         (c >= 0x2000 && c <= 0x200A) || c == 0x2028 || c == 0x2029 || c == 0x202F || c == 0x205F || c == 0x3000;
}
bool num_space(uint32_t c) { return py_isspace(c) && !(c >= 0x1C && c <= 0x1F); }

// value of a Unicode decimal digit, or -1: the category-Nd zeros, each
// followed by its nine digits
int nd_digit(uint32_t c) {
  static const uint32_t kZeros[] = {
    0x30, 0x660, 0x6F0, 0x7C0, 0x966, 0x9E6, 0xA66, 0xAE6, 0xB66, 0xBE6,
    0xC66, 0xCE6, 0xD66, 0xDE6, 0xE50, 0xED0, 0xF20, 0x1040, 0x1090, 0x17E0,
    0x1810, 0x1946, 0x19D0, 0x1A80, 0x1A90, 0x1B50, 0x1BB0, 0x1C40, 0x1C50, 0xA620,
    0xA8D0, 0xA900, 0xA9D0, 0xA9F0, 0xAA50, 0xABF0, 0xFF10, 0x104A0, 0x10D30, 0x11066,
    0x110F0, 0x11136, 0x111D0, 0x112F0, 0x11450, 0x114D0, 0x11650, 0x116C0, 0x11730, 0x118E0,
    0x11950, 0x11C50, 0x11D50, 0x11DA0, 0x11F50, 0x16A60, 0x16AC0, 0x16B50, 0x1D7CE, 0x1D7D8,
    0x1D7E2, 0x1D7EC, 0x1D7F6, 0x1E140, 0x1E2F0, 0x1E4F0, 0x1E950, 0x1FBF0,
  };
  for (uint32_t z : kZeros)
    if (c >= z && c < z + 10) return (int)(c - z);
  return -1;
}

// a number token as Python sees it, in ASCII: number whitespace stripped,
// decimal digits mapped to '0'..'9'; false if anything else is non-ASCII
bool py_number_text(const std::string& raw, std::string& out) {
  std::vector<uint32_t> cps;
  if (!utf8_decode(raw, cps)) return false;
  size_t a = 0, b = cps.size();
  while (a < b && num_space(cps[a])) ++a;
  while (b > a && num_space(cps[b - 1])) --b;
  out.clear();
  for (size_t i = a; i < b; ++i) {
    const int d = nd_digit(cps[i]);
    if (d >= 0) out += (char)('0' + d);
    else if (cps[i] < 0x80) out += (char)cps[i];
    else return false;
  }
  return true;
}

std::string py_strip(const std::string& s) {  // str.strip() on UTF-8 (unchanged if malformed)
  std::vector<uint32_t> cps;
  std::vector<size_t> at;
  if (!utf8_decode(s, cps, &at)) return s;
  size_t a = 0, b = cps.size();
  while (a < b && py_isspace(cps[a])) ++a;
  while (b > a && py_isspace(cps[b - 1])) --b;
  return s.substr(at[a], at[b] - at[a]);
}

bool is_digit(char c) { return c >= '0' && c <= '9'; }

// digits with single underscores between them, appended to `out` without
// the underscores; false if no digit at i
bool py_digits(const std::string& s, size_t& i, std::string& out) {
  if (i >= s.size() || !is_digit(s[i])) return false;
  while (i < s.size()) {
    if (is_digit(s[i])) {
      out += s[i++];
    } else if (s[i] == '_' && i + 1 < s.size() && is_digit(s[i + 1])) {
      ++i;
    } else {
      break;
    }
  }
  return true;
}

bool parse_int(const std::string& raw, int& out) {
  std::string s;
  if (!py_number_text(raw, s)) return false;
  size_t i = 0;
  bool neg = false;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  std::string d;
  if (!py_digits(s, i, d) || i != s.size()) return false;
  size_t z = 0;
  while (z + 1 < d.size() && d[z] == '0') ++z;
  d = d.substr(z);
  if (d.size() > 7) return false;  // far outside every valid width / group
  const long v = strtol(d.c_str(), nullptr, 10);
  out = (int)(neg ? -v : v);
  return true;
}

bool parse_double(const std::string& raw, double& out) {
  std::string s;
  if (!py_number_text(raw, s)) return false;
  size_t i = 0;
  std::string num;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) num += s[i++];
  std::string rest = s.substr(i);
  for (auto& c : rest) c = (char)tolower((unsigned char)c);
  if (rest == "nan" || rest == "inf" || rest == "infinity") {
    const double v = rest == "nan" ? NAN : INFINITY;
    out = (!num.empty() && num[0] == '-') ? -v : v;
    return true;
  }
  bool any = false;
  if (i < s.size() && is_digit(s[i])) any = py_digits(s, i, num);
  if (i < s.size() && s[i] == '.') {
    num += s[i++];
    if (i < s.size() && is_digit(s[i])) any = py_digits(s, i, num) || any;
  }
  if (!any) return false;
  if (i < s.size() && (s[i] == 'e' || s[i] == 'E')) {
    num += 'e';
    ++i;
    if (i < s.size() && (s[i] == '+' || s[i] == '-')) num += s[i++];
    if (!py_digits(s, i, num)) return false;
  }
  if (i != s.size()) return false;
  out = strtod(num.c_str(), nullptr);  // a plain decimal string: correctly rounded
  return true;
}

std::string py_float_repr(double v) {
  char buf[64];
  for (int p = 1; p <= 17; ++p) {
    snprintf(buf, sizeof buf, "%.*g", p, v);
    if (strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // Python repr keeps a '.0'
  return s;
}

std::string trim(const std::string& s) { return py_strip(s); }

std::vector<std::string> split(const std::string& s, char c) {
  std::vector<std::string> out;
  size_t start = 0;
  for (;;) {
    size_t p = s.find(c, start);
    out.push_back(s.substr(start, p == std::string::npos ? std::string::npos : p - start));
    if (p == std::string::npos) break;
    start = p + 1;
  }
  return out;
}

int parse_strategy(const char* text, Geo& g, double& rho, std::string& canon) {
  if (!text) return fail(KVC_ERR_CONFIG, "strategy id is NULL");
  std::string s = trim(text);
  auto seg = split(s, ';');
  if (seg.size() != 3)
    return fail(KVC_ERR_CONFIG, "strategy id must have 3 ';'-separated segments, got " + std::to_string(seg.size()));
  auto kv = [](const std::string& tok, std::string& k, std::string& v) {
    size_t p = tok.find('=');
    if (p == std::string::npos) return false;
    k = tok.substr(0, p);
    v = tok.substr(p + 1);
    return true;
  };
  std::string k, v;
  if (!kv(seg[0], k, v) || k != "t") return fail(KVC_ERR_CONFIG, "bad transform segment '" + seg[0] + "'");
  if (v == "identity") g.transform = T_IDENTITY;
  else if (v == "delta") g.transform = T_DELTA;
  else if (v == "hadamard") g.transform = T_HADAMARD;
  else if (v == "affine") g.transform = T_AFFINE;
  else return fail(KVC_ERR_CONFIG, "bad transform segment '" + seg[0] + "'");
  const std::string tname = v;

  if (!kv(seg[1], k, v) || k != "q") return fail(KVC_ERR_CONFIG, "bad quant segment '" + seg[1] + "'");
  auto qt = split(v, ',');
  std::string kind = qt[0];
  // a dict, as the reference builds it (strategy.py:84): a repeated key
  // keeps its last value
  std::vector<std::pair<std::string, std::string>> params;
  for (size_t i = 1; i < qt.size(); ++i) {
    std::string a, b;
    if (!kv(qt[i], a, b)) return fail(KVC_ERR_CONFIG, "malformed token '" + qt[i] + "' in strategy id segment '" + seg[1] + "'");
    bool seen = false;
    for (auto& p : params)
      if (p.first == a) {
        p.second = b;
        seen = true;
      }
    if (!seen) params.push_back({a, b});
  }
  auto keys_are = [&](std::initializer_list<const char*> want) {
    if (params.size() != want.size()) return false;
    for (const char* w : want) {
      int n = 0;
      for (auto& p : params) n += (p.first == w);
      if (n != 1) return false;
    }
    return true;
  };
  auto get = [&](const char* key) {
    for (auto& p : params)
      if (p.first == key) return p.second;
    return std::string();
  };
  std::string qcanon;
  g.bits = 4; g.hi = 8; g.lo = 2; rho = 0.25;
  if (kind == "uniform" || kind == "uchan") {
    if (!keys_are({"b", "g"}))
      return fail(KVC_ERR_CONFIG, kind + " quant needs exactly b and g in '" + seg[1] + "'");
    int b, gs;
    if (!parse_int(get("b"), b) || !parse_int(get("g"), gs)) return fail(KVC_ERR_CONFIG, "bad integer in '" + seg[1] + "'");
    if (gs < 1) return fail(KVC_ERR_CONFIG, "group_size must be >= 1, got " + std::to_string(gs));
    if (b < 1 || b > 8) return fail(KVC_ERR_CONFIG, "bits must be in 1..8, got " + std::to_string(b));
    g.quant = kind == "uniform" ? Q_UNIFORM : Q_UCHAN;
    g.bits = b; g.group = gs;
    qcanon = kind + ",b=" + std::to_string(b) + ",g=" + std::to_string(gs);
  } else if (kind == "mixed" || kind == "mixlayer" || kind == "mixtok") {
    if (!keys_are({"hi", "lo", "g", "rho"}))
      return fail(KVC_ERR_CONFIG, kind + " quant needs exactly hi, lo, g, rho in '" + seg[1] + "'");
    int hi, lo, gs;
    if (!parse_int(get("hi"), hi) || !parse_int(get("lo"), lo) || !parse_int(get("g"), gs) || !parse_double(get("rho"), rho))
      return fail(KVC_ERR_CONFIG, "bad number in '" + seg[1] + "'");
    if (gs < 1) return fail(KVC_ERR_CONFIG, "group_size must be >= 1, got " + std::to_string(gs));
    if (hi < 1 || hi > 8) return fail(KVC_ERR_CONFIG, "high_bits must be in 1..8, got " + std::to_string(hi));
    if (lo < 1 || lo > 8) return fail(KVC_ERR_CONFIG, "low_bits must be in 1..8, got " + std::to_string(lo));
    if (hi <= lo) return fail(KVC_ERR_CONFIG, "high_bits must exceed low_bits");
    if (!(rho >= 0.0 && rho <= 1.0)) return fail(KVC_ERR_CONFIG, "retrieval_fraction must be in [0, 1]");
    g.quant = kind == "mixed" ? Q_MIXED : (kind == "mixlayer" ? Q_MIXLAYER : Q_MIXTOK);
    g.hi = hi; g.lo = lo; g.group = gs;
    qcanon = kind + ",hi=" + std::to_string(hi) + ",lo=" + std::to_string(lo) + ",g=" + std::to_string(gs) +
             ",rho=" + py_float_repr(rho);
  } else {
    return fail(KVC_ERR_CONFIG, "unknown quant kind '" + kind + "' in '" + seg[1] + "'");
  }
  if (!kv(seg[2], k, v) || k != "c") return fail(KVC_ERR_CONFIG, "bad codec segment '" + seg[2] + "'");
  if (v == "none") g.codec = C_NONE;
  else if (v == "rle") g.codec = C_RLE;
  else if (v == "entropy") g.codec = C_ENTROPY;
  else return fail(KVC_ERR_CONFIG, "bad codec segment '" + seg[2] + "'");
  canon = "t=" + tname + ";q=" + qcanon + ";c=" + v;
  return KVC_OK;
}

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Host mirror of k_setup's stream table for a given class map.
void host_streams(const Geo& g, const uint8_t* head_classes, int n_out[1], int w[2], int64_t cnt[2]) {
  int n = 0;
  if (g.quant == Q_UNIFORM || g.quant == Q_UCHAN) {
    w[0] = g.bits; cnt[0] = g.E; n = 1;
  } else {
    int64_t hi_cnt;
    if (g.quant == Q_MIXTOK) {
      hi_cnt = g.LH * g.k_tok * g.C;
    } else {
      int64_t nhi = 0;
      for (int64_t i = 0; i < g.LH; ++i) nhi += head_classes && head_classes[i] ? 1 : 0;
      hi_cnt = nhi * g.T * g.C;
    }
    int64_t lo_cnt = g.E - hi_cnt;
    if (hi_cnt > 0) { w[n] = g.hi; cnt[n] = hi_cnt; ++n; }
    if (lo_cnt > 0) { w[n] = g.lo; cnt[n] = lo_cnt; ++n; }
  }
  n_out[0] = n;
}

}  // namespace

struct kvc_plan {
  Plan p;
};

extern "C" {

const char* kvc_last_error(void) { return g_err.c_str(); }
const char* kvc_version(void) { return "kvc 0.1 sm_100a"; }

int kvc_plan_create(kvc_plan** out, const char* strategy_id, int64_t L, int64_t H, int64_t T, int64_t C,
                    const kvc_options* opt) {
  if (!out) return fail(KVC_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  Plan p;
  memset(&p, 0, sizeof p);
  Geo& g = p.g;
  double rho = 0.25;
  std::string canon;
  int rc = parse_strategy(strategy_id, g, rho, canon);
  if (rc) return rc;
  if (L < 1 || H < 1 || T < 1 || C < 1)
    return fail(KVC_ERR_CONFIG, "all dims must be >= 1");
  g.L = L; g.H = H; g.T = T; g.C = C;
  g.LH = L * H;
  g.E = g.LH * T * C;
  g.in_dtype = opt ? opt->in_dtype : KVC_DTYPE_BF16;
  g.out_dtype = opt ? opt->out_dtype : KVC_DTYPE_BF16;
  if ((g.in_dtype != KVC_DTYPE_BF16 && g.in_dtype != KVC_DTYPE_F32) ||
      (g.out_dtype != KVC_DTYPE_BF16 && g.out_dtype != KVC_DTYPE_F32))
    return fail(KVC_ERR_CONFIG, "dtype must be KVC_DTYPE_BF16 or KVC_DTYPE_F32");
  // 2048 symbols: the adaptive model never halves inside a block for
  // alphabets <= 16 (codecs.py:227-232), which the coder exploits
  g.block = (opt && opt->block_symbols) ? opt->block_symbols : 2048;
  if (g.block <= 0 || g.block % 8) return fail(KVC_ERR_CONFIG, "block_symbols must be a positive multiple of 8");
  g.uchan = g.quant == Q_UCHAN;
  // a block that covers every symbol: rle codes the concatenated width
  // streams as one block, byte for byte the reference's whole-tensor payload
  g.rle_whole = g.codec == C_RLE && g.block >= g.E && g.E * 8 < (1ll << 31);
  g.rowlen = g.uchan ? T : C;
  if (g.rowlen % g.group)
    return fail(KVC_ERR_CONFIG, "group_size " + std::to_string(g.group) + " does not divide " +
                                    (g.uchan ? "tokens " : "channels ") + std::to_string(g.rowlen));
  if (g.transform == T_HADAMARD && (C & (C - 1)))
    return fail(KVC_ERR_CONFIG, "hadamard_over_channels needs power-of-two channels, got " + std::to_string(C));
  if (g.transform == T_HADAMARD && C > 1024) return fail(KVC_ERR_CONFIG, "hadamard supports channels <= 1024");
  if (C > 16384) return fail(KVC_ERR_CONFIG, "channels > 16384 unsupported");
  if (g.uchan && (int64_t)g.group * C * 5 > 200 * 1024)
    return fail(KVC_ERR_CONFIG, "uchan tile (group * channels) exceeds shared memory");
  if ((g.quant == Q_MIXED || g.quant == Q_MIXLAYER) && g.LH > 32768)
    return fail(KVC_ERR_CONFIG, "mixed quantization supports at most 32768 heads");
  g.G = g.rowlen / g.group;
  g.ngroups = g.E / g.group;
  g.k_tok = g.quant == Q_MIXTOK ? (int64_t)std::ceil(rho * (double)T) : 0;
  int64_t meta = 4 * g.ngroups;
  g.meta_class_off = -1;
  g.meta_affine_off = -1;
  if (g.quant == Q_MIXED || g.quant == Q_MIXLAYER) {
    g.meta_class_off = meta;
    meta += (g.LH + 7) / 8;
  }
  if (g.transform == T_AFFINE) {
    g.meta_affine_off = meta;
    meta += 4 * g.LH * C;
  }
  p.meta_bytes = meta;
  int wmax = (g.quant == Q_UNIFORM || g.quant == Q_UCHAN) ? g.bits : g.hi;
  int64_t packed_cap = (g.E * wmax + 7) / 8 + 8;
  p.max_blocks = g.codec == C_NONE ? 0 : (g.E + g.block - 1) / g.block + 1;
  if (g.codec == C_ENTROPY) p.slot_bytes = align_up(4 * g.block + 16, 16);
  else if (g.codec == C_RLE) p.slot_bytes = align_up(g.block + g.block / 128 + 16, 16);
  p.payload_cap = g.codec == C_NONE ? packed_cap : p.max_blocks * p.slot_bytes;
  p.scan_bytes = g.codec == C_NONE ? 0 : (int64_t)codec_scan_bytes(p.max_blocks);
  int64_t off = 0;
  p.ws_status = off; off += 256;
  p.ws_streams = off; off += 256;
  p.ws_heads = off; off = align_up(off + 16 * g.LH, 256);
  p.ws_packed = off; off = align_up(off + (g.codec == C_NONE ? 0 : packed_cap), 256);
  p.ws_slots = off; off = align_up(off + p.max_blocks * p.slot_bytes, 256);
  p.ws_sizes = off; off = align_up(off + 8 * (p.max_blocks + 1), 256);
  p.ws_scan = off; off = align_up(off + p.scan_bytes, 256);
  // chunked delta decode (delta128.cu)
  p.ws_delta = -1;
  if (delta128_applicable(g)) {
    p.ws_delta = off;
    off = align_up(off + delta128_ws_bytes(g), 256);
  }
  // fused Hadamard encode: the list of rows left to the exact fixup pass
  // (count + one int32 per token row at most), then a bitmap of the rows the
  // certified float32 pass hands to the float64 pass (one bit per token row)
  p.ws_fix = -1;
  if (g.transform == T_HADAMARD && fast128_applicable(g)) {
    p.ws_fix = off;
    off = align_up(off + 16 + 4 * g.LH * g.T, 16);
    off = align_up(off + 4 * ((g.LH * g.T + 31) / 32), 256);
  }
  p.ws_bytes = off;
  snprintf(p.id, sizeof p.id, "%s", canon.c_str());
  // the range coders' reciprocal tables: built (synchronously) now, so no
  // coder on any stream or inside a captured graph can run ahead of them
  if (g.codec == C_ENTROPY) {
    cudaError_t te = ensure_recip_tables();
    if (te == cudaErrorNoDevice || te == cudaErrorInsufficientDriver) {
      cudaGetLastError();  // size queries work without a GPU; launches retry and fail loudly
    } else if (te != cudaSuccess) {
      return cuda_fail(te, "range-coder tables");
    }
  }
  int dev = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&p.sm_count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    p.sm_count = 148;
  }
  kvc_plan* h = new kvc_plan;
  h->p = p;
  *out = h;
  return KVC_OK;
}

int kvc_plan_destroy(kvc_plan* plan) {
  delete plan;
  return KVC_OK;
}

const char* kvc_plan_strategy_id(const kvc_plan* plan) { return plan ? plan->p.id : ""; }

// The kernel family kvc_encode / kvc_decode dispatch to for this plan (the
// same predicates as the dispatch below), so callers can see -- and the
// Python layer warns about -- a plan that runs the generic correctness
// kernels instead of a fused head_dim-128 path.
const char* kvc_plan_encode_path(const kvc_plan* plan) {
  if (!plan) return "";
  const Geo& g = plan->p.g;
  if (fused_rc_applicable(g)) return "fused_rc";
  if (fast128_applicable(g)) {
    const int64_t box_rows = (g.in_dtype == KVC_DTYPE_F32 ? 4 : 2) * g.LH * g.T;
    if (box_rows >= (1ll << 31)) return "generic: too many token rows for a 2-D tensor map";
    if (g.transform != T_HADAMARD) return "fast128";
    // the certified float32 encoder, its float64
    // pass and the exact fixup (KVC_HADAMARD_FP64=1: the float64 encoder)
    const char* fp64 = getenv("KVC_HADAMARD_FP64");
    if (!(fp64 && atoi(fp64) != 0)) return "fast128-cert+fp64+fixup";
    return "fast128+fixup";
  }
  if (uchan128_applicable(g)) {
    if (g.in_dtype != KVC_DTYPE_BF16) return "generic: float32 input (the per-channel kernels read bf16)";
    if (g.LH * g.T >= (1ll << 31)) return "generic: 2^31 or more token rows";
    return "uchan128";
  }
  if (g.C != 128) return "generic: head_dim is not 128";
  return "generic: no fused kernel for this group / layout";
}

const char* kvc_plan_decode_path(const kvc_plan* plan) {
  if (!plan) return "";
  const Geo& g = plan->p.g;
  if (fused_rc_applicable(g)) return "fused_rc";
  if (delta128_applicable(g)) return "delta128";
  if (fast128_applicable(g)) return "fast128";
  if (uchan128_applicable(g)) return "uchan128";
  if (g.C != 128) return "generic: head_dim is not 128";
  return "generic: no fused kernel for this group / layout";
}
int64_t kvc_metadata_bytes(const kvc_plan* plan) { return plan ? plan->p.meta_bytes : -1; }
int64_t kvc_payload_capacity(const kvc_plan* plan) { return plan ? plan->p.payload_cap : -1; }
int64_t kvc_workspace_bytes(const kvc_plan* plan) { return plan ? plan->p.ws_bytes : -1; }
int64_t kvc_max_blocks(const kvc_plan* plan) { return plan ? plan->p.max_blocks : -1; }

int64_t kvc_static_payload_bytes(const kvc_plan* plan, const uint8_t* head_classes) {
  if (!plan || plan->p.g.codec != C_NONE) return -1;
  int n, w[2];
  int64_t cnt[2];
  host_streams(plan->p.g, head_classes, &n, w, cnt);
  int64_t bytes = 0;
  for (int i = 0; i < n; ++i) bytes += (cnt[i] * w[i] + 7) / 8;
  return bytes;
}

int64_t kvc_num_blocks(const kvc_plan* plan, const uint8_t* head_classes) {
  if (!plan) return -1;
  if (plan->p.g.codec == C_NONE) return 0;
  int n, w[2];
  int64_t cnt[2];
  host_streams(plan->p.g, head_classes, &n, w, cnt);
  if (plan->p.g.rle_whole) return plan->p.g.E > 0 ? 1 : 0;
  int64_t b = 0;
  for (int i = 0; i < n; ++i) b += (cnt[i] + plan->p.g.block - 1) / plan->p.g.block;
  return b;
}

static void fill_common(const Plan& p, double& hk, double& hc) {
  hc = std::sqrt((double)p.g.C);
  hk = std::ldexp(1.0 / hc, 896);
}
static void fill_common_enc(const Plan& p, double& hk, double& hc, float& hr32) {
  fill_common(p, hk, hc);
  hr32 = (float)(1.0 / hc);
}

static int encode_impl(const kvc_plan* plan, const void* kv, int paged, const int32_t* block_table,
                       int64_t page_tokens, int64_t layer_stride, const uint8_t* head_classes, void* payload,
                       void* metadata, uint64_t* block_offsets, void* workspace, void* stream) {
  if (!plan) return fail(KVC_ERR_CONFIG, "plan is NULL");
  const Plan& p = plan->p;
  const Geo& g = p.g;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!kv || !payload || !metadata || !workspace) return fail(KVC_ERR_CONFIG, "NULL buffer");
  if (g.codec != C_NONE && !block_offsets) return fail(KVC_ERR_CONFIG, "block_offsets required for rle/entropy");
  if (paged && (!block_table || page_tokens < 1 || layer_stride < 0))
    return fail(KVC_ERR_CONFIG, "paged encode needs a block table, page_tokens >= 1 and layer_stride >= 0");
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  uint8_t* meta = reinterpret_cast<uint8_t*>(metadata);
  uint32_t* status = reinterpret_cast<uint32_t*>(ws + p.ws_status);
  StreamTab* st = reinterpret_cast<StreamTab*>(ws + p.ws_streams);
  HeadEntry* heads = reinterpret_cast<HeadEntry*>(ws + p.ws_heads);
  cudaError_t e;
  if (g.quant == Q_MIXED || g.quant == Q_MIXLAYER) {
    if (!head_classes) return fail(KVC_ERR_CONFIG, "mixed_head quantization needs head labels from classify_heads");
    ClassBits cb;
    memset(&cb, 0, sizeof cb);
    for (int64_t i = 0; i < g.LH; ++i)
      if (head_classes[i]) cb.b[i >> 3] |= (uint8_t)(0x80u >> (i & 7));
    if ((e = launch_write_classmap(cb, meta + g.meta_class_off, (int)((g.LH + 7) / 8), s)) != cudaSuccess)
      return cuda_fail(e, "classmap");
  }
  if ((e = launch_setup(g, meta, st, heads, s)) != cudaSuccess) return cuda_fail(e, "setup");
  EncArgs a;
  memset(&a, 0, sizeof a);
  a.g = g;
  a.kv = kv;
  a.meta = meta;
  a.paged = paged;
  a.block_table = block_table;
  a.page_tokens = page_tokens;
  a.layer_stride = layer_stride;
  if (g.transform == T_AFFINE)
    if ((e = launch_affine_calibrate(a, s)) != cudaSuccess) return cuda_fail(e, "affine");
  if (fused_rc_applicable(g)) {
    // quantize + range code in one pass, then block offsets + gather
    FusedArgs f;
    memset(&f, 0, sizeof f);
    f.g = g;
    f.kv = kv;
    f.paged = paged;
    f.block_table = block_table;
    f.page_tokens = page_tokens;
    f.layer_stride = layer_stride;
    f.scales = reinterpret_cast<__half*>(meta);
    f.zeros = f.scales + g.ngroups;
    f.slots = ws + p.ws_slots;
    f.sizes = reinterpret_cast<uint64_t*>(ws + p.ws_sizes);
    f.slot_bytes = p.slot_bytes;
    f.max_blocks = p.max_blocks;
    f.status = status;
    for (int w = 1; w <= 8; ++w) f.rl[w] = 1.0f / (float)((1 << w) - 1);
    if ((e = launch_fused_rc_encode(f, s)) != cudaSuccess) return cuda_fail(e, "fused encode");
    CodecArgs c;
    memset(&c, 0, sizeof c);
    c.g = g;
    c.st = st;
    c.payload_out = reinterpret_cast<uint8_t*>(payload);
    c.offsets = block_offsets;
    c.slots = f.slots;
    c.sizes = f.sizes;
    c.scan_tmp = ws + p.ws_scan;
    c.scan_bytes = (size_t)p.scan_bytes;
    c.slot_bytes = p.slot_bytes;
    c.max_blocks = p.max_blocks;
    c.status = status;
    if ((e = launch_codec_finish(c, s)) != cudaSuccess) return cuda_fail(e, "codec finish");
    return KVC_OK;
  }
  a.packed = g.codec == C_NONE ? reinterpret_cast<uint8_t*>(payload) : ws + p.ws_packed;
  a.heads = heads;
  a.st = st;
  a.status = status;
  fill_common_enc(p, a.hk, a.hc, a.hr32);
  for (int w = 1; w <= 8; ++w) a.rl[w] = 1.0f / (float)((1 << w) - 1);
  const bool aligned = g.uchan ? (g.T % 8 == 0) : (g.C % 8 == 0);
  if (!aligned) {
    int64_t bytes = (g.E * ((g.quant == Q_UNIFORM || g.quant == Q_UCHAN) ? g.bits : g.hi) + 7) / 8 + 8;
    if ((e = cudaMemsetAsync(a.packed, 0, (size_t)bytes, s)) != cudaSuccess) return cuda_fail(e, "memset");
  }
  const bool fix = p.ws_fix >= 0;
  if (fix) {
    a.fix_count = reinterpret_cast<uint32_t*>(ws + p.ws_fix);
    a.fix_rows = reinterpret_cast<int32_t*>(ws + p.ws_fix + 16);
    // KVC_HADAMARD_FP64=1 keeps every row on the float64 encoder (A/B runs)
    static const bool fp64_only = getenv("KVC_HADAMARD_FP64") && atoi(getenv("KVC_HADAMARD_FP64")) != 0;
    if ((e = cudaMemsetAsync(a.fix_count, 0, 4, s)) != cudaSuccess) return cuda_fail(e, "memset");
    if (!fp64_only) {
      a.fix1_bits = reinterpret_cast<uint32_t*>(ws + align_up(p.ws_fix + 16 + 4 * g.LH * g.T, 16));
      if ((e = cudaMemsetAsync(a.fix1_bits, 0, 4 * ((g.LH * g.T + 31) / 32), s)) != cudaSuccess)
        return cuda_fail(e, "memset");
    }
  }
  if (fast128_applicable(g))
    e = launch_encode_fast128(a, p.sm_count, s);
  else if (uchan128_applicable(g))
    e = launch_encode_uchan128(a, p.sm_count, s);
  else
    e = launch_encode_generic(a, s);
  if (e != cudaSuccess) return cuda_fail(e, "encode kernel");
  if (fix && fast128_applicable(g) && g.LH * g.T < (1ll << 31)) {
    if ((e = launch_encode_fixup(a, s)) != cudaSuccess) return cuda_fail(e, "encode fixup");
  }
  if (g.codec != C_NONE) {
    CodecArgs c;
    memset(&c, 0, sizeof c);
    c.g = g;
    c.st = st;
    c.packed_in = a.packed;
    c.payload_out = reinterpret_cast<uint8_t*>(payload);
    c.offsets = block_offsets;
    c.slots = ws + p.ws_slots;
    c.sizes = reinterpret_cast<uint64_t*>(ws + p.ws_sizes);
    c.scan_tmp = ws + p.ws_scan;
    c.scan_bytes = (size_t)p.scan_bytes;
    c.slot_bytes = p.slot_bytes;
    c.max_blocks = p.max_blocks;
    c.status = status;
    if ((e = launch_codec_encode(c, p.sm_count, s)) != cudaSuccess) return cuda_fail(e, "codec encode");
  }
  return KVC_OK;
}

int kvc_encode(const kvc_plan* plan, const void* kv, const uint8_t* head_classes, void* payload, void* metadata,
               uint64_t* block_offsets, void* workspace, void* stream) {
  return encode_impl(plan, kv, 0, nullptr, 0, 0, head_classes, payload, metadata, block_offsets, workspace, stream);
}

int kvc_encode_paged(const kvc_plan* plan, const void* page_base, const int32_t* block_table, int64_t page_tokens,
                     int64_t layer_stride, const uint8_t* head_classes, void* payload, void* metadata,
                     uint64_t* block_offsets, void* workspace, void* stream) {
  return encode_impl(plan, page_base, 1, block_table, page_tokens, layer_stride, head_classes, payload, metadata,
                     block_offsets, workspace, stream);
}

static int decode_impl(const kvc_plan* plan, const void* payload, int64_t payload_bytes, const void* metadata,
                       const uint64_t* block_offsets, void* out, int paged, const int32_t* block_table,
                       int64_t page_tokens, int64_t layer_stride, void* workspace, void* stream) {
  if (!plan) return fail(KVC_ERR_CONFIG, "plan is NULL");
  const Plan& p = plan->p;
  const Geo& g = p.g;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!payload || !metadata || !workspace || !out) return fail(KVC_ERR_CONFIG, "NULL buffer");
  if (g.codec != C_NONE && !block_offsets) return fail(KVC_ERR_CONFIG, "block_offsets required for rle/entropy");
  if (paged && (!block_table || page_tokens < 1)) return fail(KVC_ERR_CONFIG, "paged decode needs a block table");
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  const uint8_t* meta = reinterpret_cast<const uint8_t*>(metadata);
  uint32_t* status = reinterpret_cast<uint32_t*>(ws + p.ws_status);
  StreamTab* st = reinterpret_cast<StreamTab*>(ws + p.ws_streams);
  HeadEntry* heads = reinterpret_cast<HeadEntry*>(ws + p.ws_heads);
  cudaError_t e;
  if ((e = launch_setup(g, meta, st, heads, s)) != cudaSuccess) return cuda_fail(e, "setup");
  if (fused_rc_applicable(g)) {
    CodecArgs c;
    memset(&c, 0, sizeof c);
    c.g = g;
    c.st = st;
    c.offsets_in = block_offsets;
    c.payload_bytes = payload_bytes;
    c.status = status;
    if ((e = launch_check_payload(c, s)) != cudaSuccess) return cuda_fail(e, "check payload");
    FusedArgs f;
    memset(&f, 0, sizeof f);
    f.g = g;
    f.scales_in = reinterpret_cast<const __half*>(meta);
    f.zeros_in = f.scales_in + g.ngroups;
    f.payload_in = reinterpret_cast<const uint8_t*>(payload);
    f.offsets_in = block_offsets;
    f.payload_bytes = payload_bytes;
    f.max_blocks = p.max_blocks;
    f.out = out;
    f.paged = paged;
    f.block_table = block_table;
    f.page_tokens = page_tokens;
    f.layer_stride = layer_stride;
    f.status = status;
    if ((e = launch_fused_rc_decode(f, s)) != cudaSuccess) return cuda_fail(e, "fused decode");
    return KVC_OK;
  }
  const uint8_t* packed = reinterpret_cast<const uint8_t*>(payload);
  CodecArgs c;
  memset(&c, 0, sizeof c);
  c.g = g;
  c.st = st;
  c.payload_in = reinterpret_cast<const uint8_t*>(payload);
  c.offsets_in = block_offsets;
  c.packed_out = ws + p.ws_packed;
  c.max_blocks = p.max_blocks;
  c.payload_bytes = payload_bytes;
  c.status = status;
  if ((e = launch_codec_decode(c, p.sm_count, s)) != cudaSuccess) return cuda_fail(e, "codec decode");
  if (g.codec != C_NONE) packed = ws + p.ws_packed;
  DecArgs a;
  memset(&a, 0, sizeof a);
  a.g = g;
  a.packed = packed;
  a.meta = meta;
  a.heads = heads;
  a.st = st;
  a.out = out;
  a.status = status;
  a.paged = paged;
  a.block_table = block_table;
  a.page_tokens = page_tokens;
  a.layer_stride = layer_stride;
  fill_common(p, a.hk, a.hc);
  if (delta128_applicable(g))
    e = launch_decode_delta128(a, p.ws_delta >= 0 ? ws + p.ws_delta : nullptr, s);
  else if (fast128_applicable(g))
    e = launch_decode_fast128(a, p.sm_count, s);
  else if (uchan128_applicable(g))
    e = launch_decode_uchan128(a, p.sm_count, s);
  else
    e = launch_decode_generic(a, s);
  if (e != cudaSuccess) return cuda_fail(e, "decode kernel");
  return KVC_OK;
}

int kvc_decode(const kvc_plan* plan, const void* payload, int64_t payload_bytes, const void* metadata,
               const uint64_t* block_offsets, void* out, void* workspace, void* stream) {
  return decode_impl(plan, payload, payload_bytes, metadata, block_offsets, out, 0, nullptr, 0, 0, workspace, stream);
}

int kvc_decode_paged(const kvc_plan* plan, const void* payload, int64_t payload_bytes, const void* metadata,
                     const uint64_t* block_offsets, void* page_base, const int32_t* block_table, int64_t page_tokens,
                     int64_t layer_stride, void* workspace, void* stream) {
  return decode_impl(plan, payload, payload_bytes, metadata, block_offsets, page_base, 1, block_table, page_tokens,
                     layer_stride, workspace, stream);
}

int kvc_block_crc32(const void* payload, const uint64_t* block_offsets, int64_t nblocks, uint32_t* crc, void* stream) {
  if (nblocks < 0) return fail(KVC_ERR_CONFIG, "nblocks < 0");
  if (nblocks == 0) return KVC_OK;
  if (!payload || !block_offsets || !crc) return fail(KVC_ERR_CONFIG, "NULL buffer");
  cudaError_t e = launch_block_crc32(reinterpret_cast<const uint8_t*>(payload), block_offsets, nblocks, crc,
                                     reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "block crc32");
  return KVC_OK;
}

int kvc_copy_device_length(void* dst, const void* src, const uint64_t* nbytes_dev, int64_t max_bytes, void* stream) {
  if (max_bytes <= 0) return KVC_OK;
  if (!dst || !src || !nbytes_dev) return fail(KVC_ERR_CONFIG, "NULL buffer");
  cudaError_t e = launch_copy_device_length(dst, src, nbytes_dev, max_bytes, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "copy");
  return KVC_OK;
}

int kvc_enable_peer_access(int device, int peer) {
  int cur = 0;
  cudaGetDevice(&cur);
  if (device == peer) return KVC_OK;
  int can = 0;
  cudaError_t e = cudaDeviceCanAccessPeer(&can, device, peer);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceCanAccessPeer");
  if (!can) return fail(KVC_ERR_CONFIG, "no peer access between these devices");
  cudaSetDevice(device);
  e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(cur);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return KVC_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return KVC_OK;
}

int kvc_sq_error(const void* a, const void* b, int64_t n, int dtype, double* sum_dev, void* stream) {
  if (n <= 0) return KVC_OK;
  if (!a || !sum_dev) return fail(KVC_ERR_CONFIG, "NULL buffer");
  if (dtype != KVC_DTYPE_BF16 && dtype != KVC_DTYPE_F32) return fail(KVC_ERR_CONFIG, "dtype must be bf16 or f32");
  if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15u) != 0)
    return fail(KVC_ERR_CONFIG, "inputs must be 16-byte aligned");
  cudaError_t e = launch_sq_error(a, b, n, dtype, sum_dev, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "sq_error");
  return KVC_OK;
}

int kvc_sq_error_partials(const void* a, const void* b, int64_t n, int dtype, double* partials, int64_t npartials,
                          void* stream) {
  if (n <= 0) return KVC_OK;
  if (!a || !partials) return fail(KVC_ERR_CONFIG, "NULL buffer");
  if (npartials < 1 || npartials > 65535) return fail(KVC_ERR_CONFIG, "npartials must be in 1..65535");
  if (dtype != KVC_DTYPE_BF16 && dtype != KVC_DTYPE_F32) return fail(KVC_ERR_CONFIG, "dtype must be bf16 or f32");
  if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15u) != 0)
    return fail(KVC_ERR_CONFIG, "inputs must be 16-byte aligned");
  cudaError_t e = launch_sq_error_partials(a, b, n, dtype, partials, npartials, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "sq_error");
  return KVC_OK;
}

int kvc_read_status(const kvc_plan* plan, void* workspace, void* stream, uint32_t* flags) {
  if (!plan || !workspace || !flags) return fail(KVC_ERR_CONFIG, "NULL argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint32_t* dev = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(workspace) + plan->p.ws_status);
  uint32_t v = 0;
  cudaError_t e = cudaMemcpyAsync(&v, dev, sizeof v, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaMemsetAsync(dev, 0, sizeof v, s);
  if (e != cudaSuccess) return cuda_fail(e, "read status");
  *flags = v;
  return KVC_OK;
}

}  // extern "C"
