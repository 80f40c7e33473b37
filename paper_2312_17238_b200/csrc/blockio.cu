// Serialized quant blocks (the reference's on-disk / wire format) straight
// into the engine: quant.deserialize_block (quant.py:364-421) restated in C++
// -- header "<BBIIBB" {version, bits, group_size, scale_group_size,
// meta_bits, ndim}, ndim u32 dims, u32 pad_count, packed codes, the zero codes
// packed meta_bits wide LSB-first (quant.py:105-128), then zero_scales,
// zero_offsets and scales as little-endian f16 -- with the reference's
// validation and messages (QuantFormatError -> MOE_ERR_FORMAT).  The parsed
// block is a moe_matrix view into the caller's buffer (zeros unpacked into
// caller scratch), loaded through moe_load_tensor / moe_load_expert.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/moeb200.h"

extern "C" int moe_engine_fail(int code, const char* msg);  // engine.cu: sets moe_last_error

namespace {

constexpr int kHeader = 12;  // struct.calcsize("<BBIIBB")

template <class T>
T rd(const uint8_t* p) {
  T v;
  memcpy(&v, p, sizeof(T));
  return v;
}

int ferr(const std::string& m) { return moe_engine_fail(MOE_ERR_FORMAT, m.c_str()); }

}  // namespace

extern "C" int moe_parse_block(const uint8_t* buf, int64_t len, moe_matrix* out,
                               uint8_t* zeros_out, int64_t zeros_cap, int64_t* n_groups_out) {
  if (!buf || !out) return moe_engine_fail(MOE_ERR_VALUE, "null argument");
  if (len < kHeader) return ferr("buffer shorter than block header");
  const int version = buf[0], bits = buf[1], meta_bits = buf[10], ndim = buf[11];
  const uint32_t g = rd<uint32_t>(buf + 2), sg = rd<uint32_t>(buf + 6);
  if (version != 1) return ferr("unsupported block version " + std::to_string(version));
  if (bits != 2 && bits != 3 && bits != 4 && bits != 16)
    return ferr("unsupported code width " + std::to_string(bits));
  int64_t off = kHeader;
  if (len < off + 4 * ndim + 4) return ferr("buffer shorter than declared shape");
  std::vector<uint32_t> shape(ndim);
  for (int i = 0; i < ndim; ++i) shape[i] = rd<uint32_t>(buf + off + 4 * i);
  off += 4 * ndim;
  const uint32_t pad = rd<uint32_t>(buf + off);
  off += 4;
  int64_t n = ndim ? 1 : 0;
  for (uint32_t d : shape) n *= d;
  memset(out, 0, sizeof(*out));
  if (ndim != 2) return moe_engine_fail(MOE_ERR_VALUE, "engine blocks must be 2-D matrices");
  out->rows = (int32_t)shape[0];
  out->cols = (int32_t)shape[1];
  out->bits = bits;
  if (bits == 16) {
    if (len - off < 2 * n) return ferr("truncated passthrough payload");
    out->codes = buf + off;
    out->codes_len = 2 * n;
    if (n_groups_out) *n_groups_out = 0;
    return MOE_OK;
  }
  const int64_t padded = n + pad;
  if (g == 0 || padded % g) return ferr("pad_count inconsistent with group size");
  const int64_t ng = padded / g;
  const int64_t nsg = (ng + (sg / g) - 1) / (sg / g);
  const int64_t nzg = (ng + sg - 1) / sg;
  const int64_t code_bytes = (padded * bits + 7) / 8;
  const int64_t zero_bytes = (ng * meta_bits + 7) / 8;
  const int64_t need = code_bytes + zero_bytes + 2 * (2 * nzg) + 2 * nsg;
  if (len - off != need)
    return ferr("payload is " + std::to_string(len - off) + " bytes, layout requires " +
                std::to_string(need));
  if (n_groups_out) *n_groups_out = ng;
  if (!zeros_out) return MOE_OK;  // size query
  if (zeros_cap < ng) return moe_engine_fail(MOE_ERR_VALUE, "zeros scratch too small");
  out->group_size = (int32_t)g;
  out->scale_group_size = (int32_t)sg;
  out->meta_bits = meta_bits;
  out->pad_count = (int32_t)pad;
  out->codes = buf + off;
  out->codes_len = code_bytes;
  off += code_bytes;
  // unpack_codes (quant.py:116-128): LSB-first bit stream, meta_bits per code
  const uint8_t* zb = buf + off;
  if (meta_bits == 8) {
    memcpy(zeros_out, zb, ng);
  } else {
    const uint32_t mask = (1u << meta_bits) - 1u;
    for (int64_t i = 0; i < ng; ++i) {
      const int64_t bit = i * meta_bits;
      uint32_t w = zb[bit >> 3];
      if (((bit & 7) + meta_bits) > 8) w |= (uint32_t)zb[(bit >> 3) + 1] << 8;
      zeros_out[i] = (uint8_t)((w >> (bit & 7)) & mask);
    }
  }
  off += zero_bytes;
  out->zeros = zeros_out;
  out->n_groups = ng;
  out->zero_scales = reinterpret_cast<const uint16_t*>(buf + off);
  off += 2 * nzg;
  out->zero_offsets = reinterpret_cast<const uint16_t*>(buf + off);
  out->n_zruns = nzg;
  off += 2 * nzg;
  out->scales = reinterpret_cast<const uint16_t*>(buf + off);
  out->n_scales = nsg;
  return MOE_OK;
}

namespace {
struct Parsed {
  moe_matrix m;
  std::vector<uint8_t> zeros;
  std::vector<uint16_t> f16;  // unaligned f16 sections copied out
};

int parse(const uint8_t* buf, int64_t len, Parsed& p) {
  int64_t ng = 0;
  int rc = moe_parse_block(buf, len, &p.m, nullptr, 0, &ng);
  if (rc) return rc;
  p.zeros.resize(ng > 0 ? ng : 1);
  rc = moe_parse_block(buf, len, &p.m, p.zeros.data(), ng, &ng);
  if (rc || p.m.bits == 16) return rc;
  // the f16 sections may sit at odd offsets in the serialized buffer
  const int64_t nz = p.m.n_zruns, ns = p.m.n_scales;
  p.f16.resize(2 * nz + ns);
  memcpy(p.f16.data(), p.m.zero_scales, 2 * nz);
  memcpy(p.f16.data() + nz, p.m.zero_offsets, 2 * nz);
  memcpy(p.f16.data() + 2 * nz, p.m.scales, 2 * ns);
  p.m.zero_scales = p.f16.data();
  p.m.zero_offsets = p.f16.data() + nz;
  p.m.scales = p.f16.data() + 2 * nz;
  return MOE_OK;
}
}  // namespace

extern "C" int moe_load_tensor_serialized(moe_engine* e, const char* name, const uint8_t* buf,
                                          int64_t len) {
  Parsed p;
  int rc = parse(buf, len, p);
  if (rc) return rc;
  if (p.m.bits == 16) {  // f16 passthrough: aligned copy of the values
    std::vector<uint16_t> v(p.m.codes_len / 2);
    memcpy(v.data(), p.m.codes, p.m.codes_len);
    p.m.codes = v.data();
    return moe_load_tensor(e, name, &p.m);
  }
  return moe_load_tensor(e, name, &p.m);
}

extern "C" int moe_load_expert_serialized(moe_engine* e, int32_t layer, int32_t expert,
                                          const uint8_t* w_gate, int64_t n_gate,
                                          const uint8_t* w_up, int64_t n_up,
                                          const uint8_t* w_down, int64_t n_down) {
  Parsed p[3];
  const uint8_t* bufs[3] = {w_gate, w_up, w_down};
  const int64_t lens[3] = {n_gate, n_up, n_down};
  for (int i = 0; i < 3; ++i) {
    int rc = parse(bufs[i], lens[i], p[i]);
    if (rc) return rc;
  }
  return moe_load_expert(e, layer, expert, &p[0].m, &p[1].m, &p[2].m);
}
