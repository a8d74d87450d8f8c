#include <algorithm>
#include <cmath>
// Prime tables: twiddles, Shoup quotients, Montgomery constants.
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <unordered_set>
#include "ctx.hpp"

namespace ctb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* get_error() { return g_err.c_str(); }

// ------------------------------------------------------------------ staged host->device uploads
// Small per-call host tables (site CSRs) are copied through a thread-local pinned ring buffer: the
// copy is stream-ordered and the call returns without synchronising; a ring region is rewritten only
// after the event recorded behind its previous copy has completed (rare: only when the ring wraps onto
// a copy still queued).  Thread-local, so the two party threads never share a region.
namespace {
struct Staging {
  char* buf = nullptr;
  size_t cap = 0, head = 0;
  struct Inflight { size_t lo, hi; cudaEvent_t ev; };
  std::vector<Inflight> inflight;
  cudaError_t drain(size_t lo, size_t hi) {  // wait for copies overlapping [lo, hi)
    cudaError_t e = cudaSuccess;
    std::vector<Inflight> keep;
    for (auto& f : inflight) {
      if (f.lo < hi && lo < f.hi) {
        if (e == cudaSuccess) e = cudaEventSynchronize(f.ev);
        cudaEventDestroy(f.ev);
      } else {
        keep.push_back(f);
      }
    }
    inflight.swap(keep);
    return e;
  }
  ~Staging() {
    drain(0, (size_t)-1);
    if (buf) cudaFreeHost(buf);  // may fail harmlessly at process teardown
  }
};
thread_local Staging g_stage;
}  // namespace

cudaError_t stage_upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (!bytes) return cudaSuccess;
  Staging& st = g_stage;
  const size_t need = (bytes + 255) & ~(size_t)255;
  cudaError_t e;
  if (need > st.cap) {
    if ((e = st.drain(0, (size_t)-1)) != cudaSuccess) return e;
    if (st.buf) cudaFreeHost(st.buf);
    st.cap = std::max<size_t>(need, (size_t)4 << 20);
    st.head = 0;
    if ((e = cudaHostAlloc((void**)&st.buf, st.cap, cudaHostAllocDefault)) != cudaSuccess) {
      st.buf = nullptr;
      st.cap = 0;
      return e;
    }
  }
  if (st.head + need > st.cap) st.head = 0;
  const size_t lo = st.head, hi = lo + need;
  if ((e = st.drain(lo, hi)) != cudaSuccess) return e;
  std::memcpy(st.buf + lo, src, bytes);
  if ((e = cudaMemcpyAsync(dst, st.buf + lo, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
  cudaEvent_t ev;
  if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaEventRecord(ev, s)) != cudaSuccess) { cudaEventDestroy(ev); return e; }
  st.inflight.push_back({lo, hi, ev});
  st.head = hi;
  return cudaSuccess;
}

static std::mutex g_attr_mu;
static std::unordered_set<const void*> g_attr_set;
bool smem_attr_done(const void* kern) {
  std::lock_guard<std::mutex> g(g_attr_mu);
  return g_attr_set.count(kern) != 0;
}
void smem_attr_mark(const void* kern) {
  std::lock_guard<std::mutex> g(g_attr_mu);
  g_attr_set.insert(kern);
}

static std::mutex g_grid_mu;
static std::unordered_map<const void*, uint32_t> g_grid;
uint32_t sm_count() {
  static const uint32_t n = [] {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (uint32_t)std::max(sms, 1);
  }();
  return n;
}

uint32_t persistent_grid(const void* kern, int threads, size_t smem) {
  {
    std::lock_guard<std::mutex> g(g_grid_mu);
    auto it = g_grid.find(kern);
    if (it != g_grid.end()) return it->second;
  }
  const int sms = (int)sm_count();
  int per_sm = 1;
  if (!smem_attr_done(kern)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_attr_mark(kern);
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const uint32_t grid = (uint32_t)(sms * per_sm);
  std::lock_guard<std::mutex> g(g_grid_mu);
  g_grid[kern] = grid;
  return grid;
}

static uint32_t bitrev(uint32_t x, uint32_t bits) {
  uint32_t y = 0;
  for (uint32_t i = 0; i < bits; ++i) { y = (y << 1) | (x & 1); x >>= 1; }
  return y;
}

// Smallest-witness primitive 2N-th root, exactly as ring._find_root_of_unity
// (ring.py:93-102): first g >= 2 whose cofactor power psi has psi^N == -1.
static bool find_psi(uint64_t p, uint32_t n, uint64_t& psi) {
  const uint64_t order = 2ull * n;
  if ((p - 1) % order != 0) return false;
  const uint64_t cof = (p - 1) / order;
  for (uint64_t g = 2; g < p && g < (1ull << 32); ++g) {
    uint64_t c = powmod(g, cof, p);
    if (powmod(c, n, p) == p - 1) { psi = c; return true; }
  }
  return false;
}

template <typename T>
static T shoup_q(uint64_t w, uint64_t p) {
  constexpr int W = 8 * sizeof(T);
  return (T)(((unsigned __int128)w << W) / p);
}

template <typename T>
static int build_typed(Base& b, uint32_t logn, std::string& err, const uint64_t* tmod,
                       const uint64_t* delta) {
  const int L = b.size();
  const uint32_t n = 1u << logn;
  constexpr int W = 8 * sizeof(T);
  std::vector<PrimeTab<T>> tabs(L);
  const int ent = shape_tw_entries((int)logn);  // entries per prime (both directions)
  const int words = tw_words<T>((int)logn);      // u32: (w, w') pairs; u64: one double per entry
  std::vector<T> tw((size_t)L * words);
  cudaError_t ce = cudaMalloc(&b.d_tw, tw.size() * sizeof(T));
  if (ce != cudaSuccess) { err = std::string("cudaMalloc twiddles: ") + cudaGetErrorString(ce); return -2; }
  ce = cudaMalloc(&b.d_tabs, sizeof(PrimeTab<T>) * (L ? L : 1));
  if (ce != cudaSuccess) { err = std::string("cudaMalloc tables: ") + cudaGetErrorString(ce); return -2; }
  T* d_tw = (T*)b.d_tw;
  for (int l = 0; l < L; ++l) {
    const uint64_t p = b.primes[l];
    uint64_t psi;
    if (!find_psi(p, n, psi)) { err = "no primitive 2N-th root of unity mod " + std::to_string(p); return -1; }
    T* f = tw.data() + (size_t)l * words;
    // powers in natural order, then scatter by bit reversal
    std::vector<uint64_t> pw(n);
    pw[0] = 1;
    for (uint32_t i = 1; i < n; ++i) pw[i] = mulmod(pw[i - 1], psi, p);
    // pass k, group B, stage i, block jb -> psi^bitrev(2^(s+i) + B*2^i + jb) at pair
    // shape_tw_pair(k, e, slot of B) with e = 2^i - 1 + jb (32-bit limbs; 64-bit limbs: tw_off(k) + e * 2^s + slot)
    for (int k = 0; k < shape_npass((int)logn); ++k) {
      const int s = shape_pass_s((int)logn, k), r = shape_pass_r((int)logn, k);
      for (int B = 0; B < (1 << s); ++B)
        for (int i = 0; i < r; ++i)
          for (int jb = 0; jb < (1 << i); ++jb) {
            const uint32_t mb = (1u << (s + i)) + ((uint32_t)B << i) + jb;
            const int ei = (1 << i) - 1 + jb, gslot = tw_group_slot((int)logn, s, r, B);
            const size_t e = sizeof(T) == 4 ? (size_t)shape_tw_pair((int)logn, k, ei, gslot)
                                            : (size_t)shape_tw_off((int)logn, k) + ((size_t)ei << s) + gslot;
            const uint64_t w = pw[bitrev(mb, logn)];
            if (sizeof(T) == 4) {
              f[2 * e] = (T)w;  f[2 * e + 1] = shoup_q<T>(w, p);
              if (ei < F64Q_NE) {  // FP64 quotient table (ntt.cuh F64Q_NE): w'/p = round(w 2^52 / p) 2^-52
                const uint64_t num = (uint64_t)((((unsigned __int128)w << 52) + p / 2) / p);
                const double wp = std::ldexp((double)num, -52);
                const size_t qe = (size_t)shape_q_index((int)logn, k, ei, gslot);
                std::memcpy(reinterpret_cast<unsigned char*>(f + 2 * ent) + 8 * qe, &wp, 8);
              }
            } else {  // 64-bit limbs run the FP64 butterflies (ntt.cuh): w CENTRED, as a double
              const double wd = w > p / 2 ? -(double)(p - w) : (double)w;
              uint64_t bw;
              std::memcpy(&bw, &wd, 8);
              f[e] = (T)bw;
            }
          }
    }
    PrimeTab<T>& t = tabs[l];
    std::memset(&t, 0, sizeof(t));
    t.p = (T)p; t.p2 = (T)(2 * p);
    t.dp = (double)p;
    t.dpinv = 1.0 / (double)p;
    T x = 1;  // Newton: p^-1 mod 2^W
    for (int it = 0; it < 7; ++it) x = (T)(x * (T)(2 - (T)p * x));
    t.pinv = x;
    const uint64_t ninv = invmod(n % p, p);
    t.ninv = (T)ninv; t.ninv_q = shoup_q<T>(ninv, p);
    const uint64_t R = (uint64_t)(((unsigned __int128)1 << W) % p);
    const uint64_t ninvr = mulmod(ninv, R, p);
    t.ninvr = (T)ninvr; t.ninvr_q = shoup_q<T>(ninvr, p);
    t.one_q = shoup_q<T>(1, p);
    t.r2 = (T)R; t.r2_q = shoup_q<T>(R, p);
    t.rr = (T)mulmod(R, R, p);
    if (sizeof(T) == 4 && p > (1ull << 25)) {
      const uint64_t c25 = (1ull << 25) % p;
      t.c25 = (T)c25; t.c25_q = shoup_q<T>(c25, p);
    }
    if (tmod) t.tmod = (T)(tmod[l] % p);
    if (delta) { t.delta = (T)(delta[l] % p); t.delta_q = shoup_q<T>(delta[l] % p, p); }
    t.fwd = d_tw + (size_t)l * words;
    t.inv = t.fwd;
  }
  ce = cudaMemcpy(b.d_tw, tw.data(), tw.size() * sizeof(T), cudaMemcpyHostToDevice);
  if (ce == cudaSuccess && L)
    ce = cudaMemcpy(b.d_tabs, tabs.data(), sizeof(PrimeTab<T>) * L, cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) { err = std::string("cudaMemcpy tables: ") + cudaGetErrorString(ce); return -2; }
  return 0;
}

int build_base(Base& b, const uint64_t* primes, int count, uint32_t logn, std::string& err,
               const uint64_t* tmod, const uint64_t* delta) {
  b.primes.assign(primes, primes + count);
  const uint32_t n = 1u << logn;
  bool small = true;
  for (uint64_t p : b.primes) {
    if (p < 3 || p % (2ull * n) != 1) { err = "prime " + std::to_string(p) + " is not 1 mod 2N"; return -1; }
    if (p >= (1ull << 50)) { err = "prime " + std::to_string(p) + " exceeds 50 bits (64-bit limbs run FP64 butterflies)"; return -1; }
    if (p >= (1ull << 30)) small = false;
  }
  b.word = small ? 4 : 8;
  return small ? build_typed<uint32_t>(b, logn, err, tmod, delta)
               : build_typed<uint64_t>(b, logn, err, tmod, delta);
}

void free_base(Base& b) {
  if (b.d_tabs) cudaFree(b.d_tabs);
  if (b.d_tw) cudaFree(b.d_tw);
  b.d_tabs = b.d_tw = nullptr;
  b.primes.clear();
}

}  // namespace ctb
