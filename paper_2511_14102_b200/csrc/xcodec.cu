// Lossless bf16 expert codec for the PCIe leg of the expert cache.
//
// Under a capped cache the decode path is bound by H2D bytes (~50 expert fetches
// per token at Phi shape, 97% of each token's time).  The copy engines move what the host store
// holds, so the store keeps every bf16 expert ENTROPY-CODED and an sm_100a kernel restores the
// exact bf16 tile images in the HBM slot as the chunks land.  Nothing about the cache decisions
// changes; the bytes the verify GEMM reads are bit-identical.
//
// Why it compresses: a bf16 weight is sign | 8-bit exponent | 7-bit mantissa.  Sign and
// mantissa are close to uniform, but the exponents of one 128x64 tile concentrate on a handful
// of values below the tile's largest one (~2.5 bits of entropy for Gaussian-like weights, which
// is what trained LLM weights look like too).  So each value is stored as its raw sign+mantissa
// byte plus a Huffman code of sym = e_max(tile) - e (sym 0..15; 16 = escape followed by the
// literal 8-bit exponent).  One canonical code (<= 12 bits) per blob, built from the blob's own
// histogram.
//
// Blob (all offsets relative to the blob start, every section 16-byte aligned):
//   [0,64)   header: u32 magic 'XCB1', u32 n_tiles, u32 hdr_bytes, u32 0, u8 code_len[17]
//   [64,..)  u32 tile_off[n_tiles + 1]           (tile_off[n_tiles] = blob bytes)
//   tiles    each: u32 e_max | mode<<8, u32 n_words, u32 0, u32 0, u16 seg_off[32]   (80 B)
//                  mode 0: u8 sm[8192] (value v's sign<<7 | mantissa, natural order)
//                          u32 words[n_words]: 32 per-lane MSB-first bit streams; lane i
//                          codes values v = 128 j + 4 i + q (j = 0..63, q = 0..3) in (j, q)
//                          order and starts at word seg_off[i]
//                  mode 1: the raw 16 KB image (a tile that would not shrink); exactly the
//                          tiles of 16464 bytes (coded tiles are always smaller)
// A tile is the 16 KB SW128 image the GEMM consumes, so decoding tile t writes bytes
// [16 KB t, 16 KB (t+1)) of the slot: the decoder needs no layout knowledge.
#include <algorithm>
#include <cstring>
#include <queue>
#include <string>
#include <vector>

#include "../../include/mspq_capi.h"
#include "common.cuh"
#include "status.h"

namespace mspq {
int set_error(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* where);

namespace {

constexpr int XC_VALS = 8192;             // values per tile (one 16 KB image)
constexpr int XC_SYMS = 17;               // 0..15 = e_max - e, 16 = escape
constexpr int XC_ESC = 16;
constexpr int XC_LUT_BITS = 12;           // longest code
constexpr int XC_THDR = 80;               // tile header bytes
constexpr int XC_RAW = XC_THDR + 2 * XC_VALS;  // 16464: raw-mode tile
constexpr int XC_SLOT = 16512;            // per-tile scratch / smem slot (>= XC_RAW + 32 slack)
constexpr uint32_t XC_MAGIC = 0x31424358u;  // "XCB1"

struct XcCode {
  uint32_t code[XC_SYMS];
  uint32_t len[XC_SYMS];
};

MSPQ_D uint32_t exp_of(uint32_t v) { return (v >> 7) & 0xFFu; }

MSPQ_D uint32_t warp_max(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Pass 1: per-tile e_max and the blob's symbol histogram (warp per tile).
__global__ void __launch_bounds__(256) k_xc_stats(const uint16_t* __restrict__ src, long long n_tiles,
                                                  uint32_t* __restrict__ emax_out,
                                                  unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[XC_SYMS];
  if (threadIdx.x < XC_SYMS) h[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long t = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t < n_tiles) {
    const uint2* s = reinterpret_cast<const uint2*>(src + t * XC_VALS);
    uint32_t em = 0;
#pragma unroll 8
    for (int j = 0; j < 64; ++j) {
      const uint2 w = s[j * 32 + lane];
      em = max(em, max(max(exp_of(w.x), exp_of(w.x >> 16)), max(exp_of(w.y), exp_of(w.y >> 16))));
    }
    em = warp_max(em);
    if (lane == 0) emax_out[t] = em;
    unsigned int c[XC_SYMS];
#pragma unroll
    for (int i = 0; i < XC_SYMS; ++i) c[i] = 0;
    for (int j = 0; j < 64; ++j) {
      const uint2 w = s[j * 32 + lane];
      const uint32_t vv[4] = {w.x & 0xFFFFu, w.x >> 16, w.y & 0xFFFFu, w.y >> 16};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t sym = min(em - exp_of(vv[q]), (uint32_t)XC_ESC);
#pragma unroll
        for (int i = 0; i < XC_SYMS; ++i) c[i] += (sym == (uint32_t)i);
      }
    }
#pragma unroll
    for (int i = 0; i < XC_SYMS; ++i) {
      unsigned int v = c[i];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v) atomicAdd(&h[i], v);
    }
  }
  __syncthreads();
  if (threadIdx.x < XC_SYMS && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

// Pass 2: encode each tile into its own XC_SLOT scratch slot (warp per tile).
__global__ void __launch_bounds__(256) k_xc_encode(const uint16_t* __restrict__ src, long long n_tiles, XcCode cc,
                                                   const uint32_t* __restrict__ emax_in, unsigned char* __restrict__ slots,
                                                   uint32_t* __restrict__ tile_bytes) {
  const int lane = threadIdx.x & 31;
  const long long t = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= n_tiles) return;
  const uint2* s = reinterpret_cast<const uint2*>(src + t * XC_VALS);
  unsigned char* out = slots + t * XC_SLOT;
  const uint32_t em = emax_in[t];
  uint32_t bits = 0;
  for (int j = 0; j < 64; ++j) {
    const uint2 w = s[j * 32 + lane];
    const uint32_t vv[4] = {w.x & 0xFFFFu, w.x >> 16, w.y & 0xFFFFu, w.y >> 16};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t sym = min(em - exp_of(vv[q]), (uint32_t)XC_ESC);
      bits += cc.len[sym] + (sym == XC_ESC ? 8u : 0u);
    }
  }
  const uint32_t words = (bits + 31) >> 5;
  uint32_t off = words;  // inclusive scan -> exclusive
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, off, o);
    if (lane >= o) off += v;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, off, 31);
  off -= words;
  const uint32_t size = (XC_THDR + XC_VALS + 4 * total + 15) & ~15u;
  uint32_t* hdr = reinterpret_cast<uint32_t*>(out);
  if (size >= (uint32_t)XC_RAW) {  // would not shrink: raw image (the decoder keys on the size)
    if (lane == 0) {
      hdr[0] = em | (1u << 8);
      hdr[1] = 0;
      hdr[2] = hdr[3] = 0;
    }
    const uint4* s4 = reinterpret_cast<const uint4*>(src + t * XC_VALS);
    uint4* d4 = reinterpret_cast<uint4*>(out + XC_THDR);
    for (int i = lane; i < 2 * XC_VALS / 16; i += 32) d4[i] = s4[i];
    if (lane == 0) tile_bytes[t] = XC_RAW;
    return;
  }
  if (lane == 0) {
    hdr[0] = em;
    hdr[1] = total;
    hdr[2] = hdr[3] = 0;
  }
  reinterpret_cast<uint16_t*>(out + 16)[lane] = (uint16_t)off;
  uint32_t* wp = reinterpret_cast<uint32_t*>(out + XC_THDR + XC_VALS) + off;
  uint64_t acc = 0;
  int nacc = 0;
  for (int j = 0; j < 64; ++j) {
    const uint2 w = s[j * 32 + lane];
    const uint32_t vv[4] = {w.x & 0xFFFFu, w.x >> 16, w.y & 0xFFFFu, w.y >> 16};
    uint32_t smw = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t v = vv[q], e = exp_of(v);
      smw |= (((v >> 8) & 0x80u) | (v & 0x7Fu)) << (8 * q);
      const uint32_t sym = min(em - e, (uint32_t)XC_ESC);
      uint32_t c = cc.code[sym], l = cc.len[sym];
      if (sym == XC_ESC) {
        c = (c << 8) | e;
        l += 8;
      }
      acc = (acc << l) | c;
      nacc += (int)l;
      if (nacc >= 32) {
        nacc -= 32;
        *wp++ = (uint32_t)(acc >> nacc);
      }
    }
    *reinterpret_cast<uint32_t*>(out + XC_THDR + 128 * j + 4 * lane) = smw;
  }
  if (nacc > 0) *wp = (uint32_t)(acc << (32 - nacc));
  if (lane == 0) tile_bytes[t] = size;
}

// Pass 3: pack the slots at their final offsets.
__global__ void k_xc_compact(const unsigned char* __restrict__ slots, const uint32_t* __restrict__ tile_off,
                             long long n_tiles, unsigned char* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long t = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= n_tiles) return;
  const uint32_t n16 = (tile_off[t + 1] - tile_off[t]) >> 4;
  const uint4* s = reinterpret_cast<const uint4*>(slots + t * XC_SLOT);
  uint4* d = reinterpret_cast<uint4*>(out + tile_off[t]);
  for (uint32_t i = lane; i < n16; i += 32) d[i] = s[i];
}


// Decode tiles [t0, t1) of a blob into dst (tile t -> dst + 8192 t).  One tile per warp at a
// time, 8 warps per CTA, 4 CTAs per SM: the per-lane decode is a serial dependency chain, so
// throughput comes from warps in flight, and only the 16 KB code table lives in shared memory.
// Every lane reads its own bit stream straight from the blob (L1-cached: one 128 B line feeds
// ~500 of its values) with a 12-bit window into a MULTI-SYMBOL table (up to 4 codes per lookup;
// ~2 bits per code for these weights), queues the exponents in a register FIFO and, 4 at a
// time, joins them with their sign|mantissa bytes (coalesced 128 B per warp, loaded one step
// ahead) into 8 bytes of bf16 (one 256 B store per warp).  Escape-class codes (sym 15, 16)
// carry (len, sym) in the table instead.  Raw tiles are copied through.
constexpr int XC_WARPS = 8;
__global__ void __launch_bounds__(XC_WARPS * 32, 4) k_xc_decode(const unsigned char* __restrict__ blob, int t0,
                                                                int t1, uint16_t* __restrict__ dst) {
  __shared__ uint32_t lut[1 << XC_LUT_BITS];  // 16 KB
  __shared__ uint16_t lut1[1 << XC_LUT_BITS];  // 8 KB single-code table (builds lut)
  __shared__ uint32_t codes[XC_SYMS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint8_t* lens = blob + 16;
  if (threadIdx.x == 0) {  // canonical code assignment in (len, sym) order
    uint32_t code = 0;
    for (uint32_t l = 1; l <= (uint32_t)XC_LUT_BITS; ++l) {
      for (int s = 0; s < XC_SYMS; ++s)
        if (lens[s] == l) codes[s] = code++;
      code <<= 1;
    }
  }
  __syncthreads();
  for (int s = 0; s < XC_SYMS; ++s) {
    const uint32_t l = lens[s];
    if (l == 0 || l > (uint32_t)XC_LUT_BITS) continue;
    const uint32_t lo = codes[s] << (XC_LUT_BITS - l), n = 1u << (XC_LUT_BITS - l);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) lut1[lo + i] = (uint16_t)((l << 8) | s);
  }
  __syncthreads();
  for (uint32_t w = threadIdx.x; w < (1u << XC_LUT_BITS); w += blockDim.x) {
    uint32_t ent = 0, used = 0;
    for (int n = 0; n < 4; ++n) {
      const uint32_t e1 = lut1[((w << (32 - XC_LUT_BITS)) << used) >> (32 - XC_LUT_BITS)];
      const uint32_t l = e1 >> 8, sy = e1 & 0xFFu;
      if (sy >= 15 || used + l > (uint32_t)XC_LUT_BITS) {
        if (n == 0) ent = e1;  // escape class: (len << 8) | sym, cum0 nibble = 0
        break;
      }
      used += l;
      ent |= (sy << (4 * n)) | (used << (16 + 4 * n));
    }
    lut[w] = ent;
  }
  __syncthreads();
  const uint32_t* toff = reinterpret_cast<const uint32_t*>(blob + 64);
  for (int t = t0 + blockIdx.x * XC_WARPS + warp; t < t1; t += gridDim.x * XC_WARPS) {
    const uint32_t off = __ldg(toff + t), bytes = __ldg(toff + t + 1) - off;
    const unsigned char* tb = blob + off;
    uint16_t* d = dst + (long long)t * XC_VALS;
    if (bytes == (uint32_t)XC_RAW) {  // raw tile
      const uint4* s4 = reinterpret_cast<const uint4*>(tb + XC_THDR);
      uint4* d4 = reinterpret_cast<uint4*>(d);
      for (int k = lane; k < 2 * XC_VALS / 16; k += 32) d4[k] = __ldg(s4 + k);
      continue;
    }
    const uint32_t em = __ldg(reinterpret_cast<const uint32_t*>(tb)) & 0xFFu, em4 = em * 0x01010101u;
    const uint32_t* ws = reinterpret_cast<const uint32_t*>(tb + XC_THDR + XC_VALS) +
                         __ldg(reinterpret_cast<const uint16_t*>(tb + 16) + lane);
    const uint32_t* smg = reinterpret_cast<const uint32_t*>(tb + XC_THDR) + lane;
    // the lane's bit stream: two live words plus two loaded ahead (each refill's L2 latency used to
    // stall the next word crossing)
    // (reads stay inside the tile's stream area: words past its end come back as 0)
    const uint32_t* wbase = reinterpret_cast<const uint32_t*>(tb + XC_THDR + XC_VALS);
    const int wend = (int)__ldg(reinterpret_cast<const uint32_t*>(tb) + 1) - (int)(ws - wbase);
    auto wload = [&](int i) { return i < wend ? __ldg(ws + i) : 0u; };
    uint32_t cur = wload(0), nxt = wload(1), q2 = wload(2), q3 = wload(3);
    int wi = 4, bp = 0, cnt = 0;
    uint64_t fifo = 0;
    uint2* d2 = reinterpret_cast<uint2*>(d) + lane;
    // sign|mantissa words: each step j reads a new 128 B line, so they are fetched 8 steps ahead
    // (two 8-word register blocks) -- one step ahead left ~64 L2 round trips per tile exposed
    uint32_t smb0[8], smb1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) smb0[u] = __ldg(smg + 32 * u);
#pragma unroll 1
    for (int jb = 0; jb < 64; jb += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) smb1[u] = jb + 8 < 64 ? __ldg(smg + 32 * (jb + 8 + u)) : 0u;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
      const int j = jb + u;
      const uint32_t smw = smb0[u];
      while (cnt < 4) {
        const uint32_t win = __funnelshift_l(nxt, cur, bp);
        const uint32_t ent = lut[win >> (32 - XC_LUT_BITS)];
        uint32_t adv, add;
        int m;
        if ((ent & 0xF0000u) == 0) {  // escape-class code
          adv = (ent >> 8) & 0xFFu;
          const uint32_t sy = ent & 0xFFu;
          add = em - sy;
          if (sy == (uint32_t)XC_ESC) {
            add = (win << adv) >> 24;
            adv += 8;
          }
          m = 1;
        } else {
          m = 1 + (((ent >> 20) & 15u) != 0) + (((ent >> 24) & 15u) != 0) + ((ent >> 28) != 0);
          const uint32_t x = ent & 0xFFFFu;
          add = em4 - ((x & 0xFu) | ((x & 0xF0u) << 4) | ((x & 0xF00u) << 8) | ((x & 0xF000u) << 12));
          add &= 0xFFFFFFFFu >> (32 - 8 * m);
          adv = (ent >> (12 + 4 * m)) & 15u;
        }
        fifo |= (uint64_t)add << (8 * cnt);
        cnt += m;
        bp += (int)adv;
        if (bp >= 32) {
          bp -= 32;
          cur = nxt;
          nxt = q2;
          q2 = q3;
          q3 = wload(wi++);
        }
      }
      const uint32_t ew = (uint32_t)fifo;
      fifo >>= 32;
      cnt -= 4;
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t smb = (smw >> (8 * q)) & 0xFFu, e = (ew >> (8 * q)) & 0xFFu;
        o[q] = ((smb & 0x80u) << 8) | (e << 7) | (smb & 0x7Fu);
      }
      d2[32 * j] = make_uint2(o[0] | (o[1] << 16), o[2] | (o[3] << 16));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) smb0[u] = smb1[u];
    }
  }
}


// Length-limited Huffman code lengths: plain Huffman, then flatten the counts until the
// longest code fits XC_LUT_BITS.  Every symbol gets a code (count >= 1).
void huff_lengths(const unsigned long long* cnt_in, uint8_t* len) {
  std::vector<unsigned long long> cnt(cnt_in, cnt_in + XC_SYMS);
  for (auto& c : cnt) c = std::max<unsigned long long>(c, 1);
  for (;;) {
    struct Node {
      unsigned long long w;
      int id;
      bool operator>(const Node& o) const { return w != o.w ? w > o.w : id > o.id; }
    };
    std::priority_queue<Node, std::vector<Node>, std::greater<Node>> pq;
    std::vector<int> parent(2 * XC_SYMS, -1);
    for (int i = 0; i < XC_SYMS; ++i) pq.push({cnt[i], i});
    int next = XC_SYMS;
    while (pq.size() > 1) {
      Node a = pq.top();
      pq.pop();
      Node b = pq.top();
      pq.pop();
      parent[a.id] = parent[b.id] = next;
      pq.push({a.w + b.w, next++});
    }
    int maxl = 0;
    for (int i = 0; i < XC_SYMS; ++i) {
      int l = 0;
      for (int p = i; parent[p] >= 0; p = parent[p]) ++l;
      len[i] = (uint8_t)l;
      maxl = std::max(maxl, l);
    }
    if (maxl <= XC_LUT_BITS) return;
    for (auto& c : cnt) c = (c >> 1) | 1;
  }
}

XcCode canonical(const uint8_t* len) {
  XcCode cc{};
  uint32_t code = 0;
  for (uint32_t l = 1; l <= (uint32_t)XC_LUT_BITS; ++l) {
    for (int s = 0; s < XC_SYMS; ++s)
      if (len[s] == l) {
        cc.code[s] = code++;
        cc.len[s] = l;
      }
    code <<= 1;
  }
  return cc;
}

size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
size_t hdr_bytes(long long n) { return 64 + (((size_t)(n + 1) * 4 + 15) & ~size_t(15)); }

}  // namespace
}  // namespace mspq

using namespace mspq;

extern "C" {

long long mspq_xc_max_blob_bytes(long long n_tiles) { return (long long)(hdr_bytes(n_tiles) + (size_t)n_tiles * XC_RAW); }
long long mspq_xc_scratch_bytes(long long n_tiles) {
  return (long long)(al256(XC_SYMS * 8) + al256((size_t)n_tiles * 4) * 2 + (size_t)n_tiles * XC_SLOT + 256);
}

int mspq_xc_encode(const void* tiles, long long n_tiles, void* scratch, void* out, long long out_cap,
                   long long* out_bytes, void* stream) {
  if (n_tiles < 1 || n_tiles > (1 << 24)) return set_error(MSPQ_ERR_SHAPE_MISMATCH, "xc_encode: bad tile count");
  if (((uintptr_t)tiles | (uintptr_t)out | (uintptr_t)scratch) & 255)
    return set_error(MSPQ_ERR_SHAPE_MISMATCH, "xc_encode: buffers must be 256-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* sb = (unsigned char*)scratch;
  unsigned long long* hist = (unsigned long long*)sb;
  uint32_t* emax = (uint32_t*)(sb + al256(XC_SYMS * 8));
  uint32_t* tbytes = (uint32_t*)((unsigned char*)emax + al256((size_t)n_tiles * 4));
  unsigned char* slots = (unsigned char*)tbytes + al256((size_t)n_tiles * 4);
  const int grid = (int)((n_tiles + 7) / 8);
  cudaError_t e = cudaMemsetAsync(hist, 0, XC_SYMS * 8, st);
  if (e != cudaSuccess) return cuda_status(e, "xc hist memset");
  k_xc_stats<<<grid, 256, 0, st>>>((const uint16_t*)tiles, n_tiles, emax, hist);
  unsigned long long h[XC_SYMS];
  e = cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e, "xc_stats");
  uint8_t len[32] = {0};
  huff_lengths(h, len);
  const XcCode cc = canonical(len);
  k_xc_encode<<<grid, 256, 0, st>>>((const uint16_t*)tiles, n_tiles, cc, emax, slots, tbytes);
  std::vector<uint32_t> off((size_t)n_tiles + 1);
  e = cudaMemcpyAsync(off.data() + 1, tbytes, (size_t)n_tiles * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e, "xc_encode");
  const size_t hb = hdr_bytes(n_tiles);
  unsigned long long run = hb;
  off[0] = (uint32_t)hb;
  for (long long t = 1; t <= n_tiles; ++t) {
    run += off[t];
    off[t] = (uint32_t)run;
  }
  if (run > 0xFFFFFFFFull) return set_error(MSPQ_ERR_SHAPE_MISMATCH, "xc_encode: blob exceeds 4 GB");
  if ((long long)run > out_cap) return set_error(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "xc_encode: output too small");
  std::vector<unsigned char> head(hb, 0);
  const uint32_t h4[4] = {XC_MAGIC, (uint32_t)n_tiles, (uint32_t)hb, 0};
  memcpy(head.data(), h4, 16);
  memcpy(head.data() + 16, len, XC_SYMS);
  memcpy(head.data() + 64, off.data(), ((size_t)n_tiles + 1) * 4);
  e = cudaMemcpyAsync(out, head.data(), hb, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_status(e, "xc header");
  k_xc_compact<<<grid, 256, 0, st>>>(slots, (const uint32_t*)((unsigned char*)out + 64), n_tiles, (unsigned char*)out);
  e = cudaStreamSynchronize(st);  // head[] is pageable and goes out of scope
  if (e != cudaSuccess) return cuda_status(e, "xc_compact");
  *out_bytes = (long long)run;
  return MSPQ_OK;
}

int mspq_xc_decode(const void* blob, int tile0, int tile1, void* dst, int n_ctas, void* stream) {
  if (tile0 < 0 || tile1 < tile0) return set_error(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "xc_decode: bad tile range");
  if (tile1 == tile0) return MSPQ_OK;
  const int need = (tile1 - tile0 + XC_WARPS - 1) / XC_WARPS;
  const int grid = std::max(1, std::min(n_ctas > 0 ? n_ctas : 32, need));
  // decodes run beside the verify GEMM (K3, ~57 KB smem per CTA): ask for the max-shared carveout
  // so an SM holding a decode CTA is not configured with too little shared memory to co-host K3
  static bool carve = false;
  if (!carve) {
    cudaFuncSetAttribute(k_xc_decode, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    carve = true;
  }
  k_xc_decode<<<grid, XC_WARPS * 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>((const unsigned char*)blob, tile0,
                                                                                  tile1, (uint16_t*)dst);
  return cuda_status(cudaGetLastError(), "xc_decode");
}

}  // extern "C"
