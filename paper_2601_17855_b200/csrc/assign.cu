// Batched policy operator: many independent assign() calls
// (policies.hpp:372-382), one warp per call -- fcfs (:100-114), jsq
// (:118-138), bfio-greedy (:269-370) and bfio-exact (:182-259, the
// lexicographic-first minimum of the exhaustive search, split over the 32
// lanes by search-tree prefix). Inputs are the reference's previews and views
// as exact integers (the host checks every value is an integer in [0, 2^31)).
#include <cuda_runtime.h>

#include <cstdint>

#include "assign.cuh"

namespace bfsim {
namespace {

#define AFULL 0xffffffffu

__device__ __forceinline__ unsigned lanemask_lt_a() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint64_t wmin64(uint64_t v) {
  const uint32_t hi = __reduce_min_sync(AFULL, static_cast<uint32_t>(v >> 32));
  const uint32_t lo =
      __reduce_min_sync(AFULL, static_cast<uint32_t>(v >> 32) == hi ? static_cast<uint32_t>(v) : 0xFFFFFFFFu);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

struct Warp {
  const AssignParams& P;
  const bfsim_assign_call_t& c;
  int lane, n, G, H, U;
  const int64_t* pv;   // [n][H+1]
  const int64_t* fut;  // [G][H+1]
  const int32_t* caps;
  const int32_t* cnt;
  int32_t* choice;  // [n] worker or G (workspace)
};

// Pairs (i, choice[i]) for choice[i] < G, in waiting order (the reference's
// order for every policy: natural for fcfs/jsq/exact, sorted for greedy).
__device__ int64_t emit_pairs(const Warp& w) {
  int64_t out = 0;
  for (int base = 0; base < w.n; base += 32) {
    const int i = base + w.lane;
    const bool has = i < w.n && w.choice[i] < w.G;
    const unsigned m = __ballot_sync(AFULL, has);
    if (has) {
      const int64_t k = out + __popc(m & lanemask_lt_a());
      w.P.pairs[w.c.pair_offset + 2 * k] = i;
      w.P.pairs[w.c.pair_offset + 2 * k + 1] = w.choice[i];
    }
    out += __popc(m);
  }
  return out;
}

// fcfs: argmax cap, lowest index; jsq: argmin count over cap > 0, lowest index.
__device__ void fifo(const Warp& w, bool jsq) {
  int cap = w.lane < w.G ? w.caps[w.lane] : 0;
  int cnt = w.lane < w.G ? w.cnt[w.lane] : 0;
  long long free_total = __reduce_add_sync(AFULL, static_cast<unsigned>(cap > 0 ? cap : 0));
  for (int i = w.lane; i < w.n; i += 32) w.choice[i] = w.G;
  __syncwarp();
  for (int i = 0; i < w.n; ++i) {
    uint32_t key;
    if (!jsq) {
      if (free_total <= 0) break;
      // largest cap first (caps < 2^20), then lowest index
      key = w.lane < w.G ? (static_cast<uint32_t>((1 << 20) - 1 - cap) << 5) | w.lane : 0xFFFFFFFFu;
    } else {
      key = (w.lane < w.G && cap > 0) ? (static_cast<uint32_t>(cnt) << 5) | w.lane : 0xFFFFFFFFu;
    }
    const uint32_t km = __reduce_min_sync(AFULL, key);
    if (km == 0xFFFFFFFFu) break;
    const int best = static_cast<int>(km & 31u);
    if (w.lane == best) {
      --cap;
      ++cnt;
      w.choice[i] = best;
    }
    --free_total;
  }
  __syncwarp();
}

// bfio_assign_greedy (policies.hpp:269-370) on arbitrary integer previews.
__device__ void greedy(const Warp& w, int32_t* sorted, int32_t* order, int64_t* F, int64_t* wrow) {
  const int n = w.n, G = w.G, H = w.H, lane = w.lane;
  const int H1 = H + 1;
  for (int i = lane; i < n; i += 32) w.choice[i] = G;
  int cap = lane < G ? w.caps[lane] : 0;
  for (int h = 0; h <= H; ++h)
    if (lane < G) F[h * 32 + lane] = w.fut[lane * H1 + h];
  __syncwarp();
  const int U = w.U;
  int nsel = 0;
  if (n == U) {
    for (int i = lane; i < n; i += 32) order[i] = i;
    nsel = n;
  } else {
    // stable sort of the waiting list by w0 ascending (:288-291)
    for (int i = lane; i < n; i += 32) {
      const int64_t wi = w.pv[i * H1];
      int r = 0;
      for (int j = 0; j < n; ++j) {
        const int64_t wj = w.pv[j * H1];
        r += (wj < wi || (wj == wi && j < i)) ? 1 : 0;
      }
      sorted[r] = i;
    }
    __syncwarp();
    // water filling (:292-323); used entries are marked by sorted[j] = -1 - i
    int64_t load = lane < G ? F[lane] : 0;
    int fr = cap;
    int64_t target = static_cast<int64_t>(
        __reduce_max_sync(AFULL, static_cast<uint32_t>(lane < G ? load : 0)));
    for (int left = U; left > 0; --left) {
      const uint64_t key = (lane < G && fr > 0) ? (static_cast<uint64_t>(load) << 5) | lane : ~0ull;
      const uint64_t km = wmin64(key);
      if (km == ~0ull) break;
      const int g = static_cast<int>(km & 31u);
      const int64_t lg = static_cast<int64_t>(km >> 5);
      const int64_t deficit = target - lg;
      int pick = -1;
      for (int base = ((n + 31) & ~31) - 32; base >= 0 && pick < 0; base -= 32) {
        const int j = base + lane;
        const bool ok = j < n && sorted[j] >= 0 && w.pv[sorted[j] * H1] <= deficit;
        const unsigned m = __ballot_sync(AFULL, ok);
        if (m) pick = base + 31 - __clz(m);
      }
      for (int base = 0; base < n && pick < 0; base += 32) {
        const int j = base + lane;
        const unsigned m = __ballot_sync(AFULL, j < n && sorted[j] >= 0);
        if (m) pick = base + __ffs(m) - 1;
      }
      if (pick < 0) break;
      const int i = sorted[pick];
      __syncwarp();
      if (lane == 0) {
        sorted[pick] = -1 - i;
        order[nsel] = i;
      }
      ++nsel;
      const int64_t w0 = w.pv[i * H1];
      if (lane == g) {
        load += w0;
        --fr;
      }
      const int64_t nl = lg + w0;
      target = nl > target ? nl : target;
      __syncwarp();
    }
  }
  __syncwarp();
  // stable sort of the selection by w0 descending (:324-326): rank, then scatter
  for (int q = lane; q < nsel; q += 32) {
    const int i = order[q];
    const int64_t wi = w.pv[i * H1];
    int r = 0;
    for (int p = 0; p < nsel; ++p) {
      const int64_t wp = w.pv[order[p] * H1];
      r += (wp > wi || (wp == wi && p < q)) ? 1 : 0;
    }
    sorted[r] = i;  // `sorted` is free again
  }
  __syncwarp();
  // placement (:339-367), restated as argmin over cap > 0 of
  // (sum_h max(M_h, F_h[g] + w_h), F_0[g], g) with M_h the max over all
  // workers (the horizon cost up to a g-independent term)
  for (int q = 0; q < nsel; ++q) {
    const int i = sorted[q];
    for (int h = lane; h <= H; h += 32) wrow[h] = w.pv[i * H1 + h];
    __syncwarp();
    uint64_t cost = ~0ull;
    if (lane < G && cap > 0) {
      cost = 0;
      for (int h = 0; h <= H; ++h) {
        int64_t m = 0;
        for (int g = 0; g < G; ++g) m = F[h * 32 + g] > m ? F[h * 32 + g] : m;
        const int64_t v = F[h * 32 + lane] + wrow[h];
        cost += static_cast<uint64_t>(v > m ? v : m);
      }
    }
    const uint64_t cmin = wmin64(cost);
    if (cmin == ~0ull) break;
    const uint64_t k2 = (cost == cmin) ? (static_cast<uint64_t>(F[lane < G ? lane : 0]) << 5) | lane : ~0ull;
    const int best = static_cast<int>(wmin64(k2) & 31u);
    __syncwarp();
    for (int h = lane; h <= H; h += 32) F[h * 32 + best] += wrow[h];
    if (lane == best) --cap;
    if (lane == 0) w.choice[i] = best;
    __syncwarp();
  }
  __syncwarp();
}

// bfio-exact (ExactSearch, policies.hpp:182-233): every feasible assignment
// vector in lexicographic order (workers 0..G-1, then unassigned); the first
// minimum of horizon_cost wins; more than `limit` full allocations throws.
// Lanes take search-tree prefixes p = lane, lane + 32, ... (prefix order is
// lexicographic), run the sequential search below each, and the warp keeps
// the smallest (cost, p).
__device__ void exact(const Warp& w, int32_t* lchoice, int32_t* bchoice, int64_t* L, int32_t* lcap,
                      int32_t* opt, int64_t limit, double* cost_out, int32_t* status) {
  const int n = w.n, G = w.G, H = w.H, lane = w.lane, U = w.U;
  const int H1 = H + 1;
  int d = 0;
  long long P = 1;
  while (d < n && P < 64) {
    P *= (G + 1);
    ++d;
  }
  long long leaves = 0;
  bool found = false;
  int64_t best = 0;
  long long bestp = -1;
  auto hcost = [&]() -> int64_t {
    int64_t j = 0;
    for (int h = 0; h <= H; ++h) {
      int64_t mx = 0, sum = 0;
      for (int g = 0; g < G; ++g) {
        const int64_t x = L[h * G + g];
        mx = x > mx ? x : mx;
        sum += x;
      }
      j += static_cast<int64_t>(G) * mx - sum;
    }
    return j;
  };
  for (long long p = lane; p < P && leaves <= limit; p += 32) {
    for (int g = 0; g < G; ++g) lcap[g] = w.caps[g];
    for (int h = 0; h <= H; ++h)
      for (int g = 0; g < G; ++g) L[h * G + g] = w.fut[g * H1 + h];
    // walk the prefix
    long long rest = p, div = P;
    int assigned = 0;
    bool ok = true;
    for (int i = 0; i < d && ok; ++i) {
      if (assigned + (n - i) < U) ok = false;
      div /= (G + 1);
      const int ch = static_cast<int>(rest / div);
      rest %= div;
      if (!ok) break;
      if (ch < G) {
        if (lcap[ch] <= 0 || assigned >= U) {
          ok = false;
          break;
        }
        --lcap[ch];
        ++assigned;
        for (int h = 0; h <= H; ++h) L[h * G + ch] += w.pv[i * H1 + h];
      }
      lchoice[i] = ch;
    }
    if (!ok) continue;
    // sequential search below the prefix, iterative: opt[i] is the option
    // applied at level i (G = unassigned, tried last)
    auto apply = [&](int i, int g) {
      lchoice[i] = g;
      if (g < G) {
        --lcap[g];
        ++assigned;
        for (int h = 0; h <= H; ++h) L[h * G + g] += w.pv[i * H1 + h];
      }
    };
    auto undo = [&](int i, int g) {
      if (g < G) {
        ++lcap[g];
        --assigned;
        for (int h = 0; h <= H; ++h) L[h * G + g] -= w.pv[i * H1 + h];
      }
    };
    auto first_from = [&](int g) {  // next worker option >= g, else unassigned
      while (g < G && !(lcap[g] > 0 && assigned < U)) ++g;
      return g;
    };
    int i = d;
    bool down = true;
    while (leaves <= limit) {
      if (down) {
        if (assigned + (n - i) < U || i == n) {
          if (i == n && assigned == U) {
            ++leaves;
            const int64_t c = hcost();
            if (!found || c < best) {  // the first minimum in enumeration order
              found = true;
              best = c;
              bestp = p;
              for (int t = 0; t < n; ++t) bchoice[t] = lchoice[t];
            }
          }
          down = false;
          if (--i < d) break;
          continue;
        }
        opt[i] = first_from(0);
        apply(i, opt[i]);
        ++i;
      } else {
        const int g = opt[i];
        undo(i, g);
        if (g == G) {
          if (--i < d) break;
          continue;
        }
        opt[i] = first_from(g + 1);
        apply(i, opt[i]);
        ++i;
        down = true;
      }
    }
  }
  // warp: total leaves, then the smallest (cost, prefix)
  unsigned long long tot = leaves;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(AFULL, tot, off);
  if (static_cast<long long>(tot) > limit) {
    if (lane == 0) *status = BFSIM_ELIMIT;
    for (int t = lane; t < n; t += 32) w.choice[t] = G;
    __syncwarp();
    return;
  }
  const uint64_t ck = found ? static_cast<uint64_t>(best) : ~0ull;
  const uint64_t cm = wmin64(ck);
  const uint64_t pk = (found && ck == cm) ? static_cast<uint64_t>(bestp) : ~0ull;
  const uint64_t pm = wmin64(pk);
  const unsigned wm = __ballot_sync(AFULL, found && ck == cm && static_cast<uint64_t>(bestp) == pm);
  const int winner = wm ? __ffs(wm) - 1 : -1;
  if (lane == winner)
    for (int t = 0; t < n; ++t) w.choice[t] = bchoice[t];
  if (lane == 0 && winner < 0)
    for (int t = 0; t < n; ++t) w.choice[t] = G;
  __syncwarp();
  if (winner >= 0) {
    if (lane == winner) *cost_out = static_cast<double>(best);
  } else if (lane == 0) {
    // no feasible allocation: horizon_cost of the current views
    for (int h = 0; h <= H; ++h)
      for (int g = 0; g < G; ++g) L[h * G + g] = w.fut[g * H1 + h];
    *cost_out = static_cast<double>(hcost());
  }
}

__global__ void __launch_bounds__(32) assign_kernel(AssignParams P) {
  const int call = blockIdx.x;
  if (call >= P.n_calls) return;
  const bfsim_assign_call_t& c = P.calls[call];
  const int lane = threadIdx.x & 31;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* ws = P.ws + static_cast<size_t>(call) * P.ws_stride;
  Warp w{P, c, lane, c.n_waiting, c.workers, c.horizon, 0, P.previews + c.preview_offset,
         P.futures + c.future_offset, P.caps + c.worker_offset, P.counts + c.worker_offset,
         reinterpret_cast<int32_t*>(ws)};
  long long capsum = 0;
  for (int g = lane; g < w.G; g += 32) capsum += w.caps[g] > 0 ? w.caps[g] : 0;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) capsum += __shfl_xor_sync(AFULL, capsum, off);
  w.U = static_cast<int>(w.n < capsum ? w.n : capsum);
  if (lane == 0) {
    P.status[call] = BFSIM_OK;
    P.cost[call] = 0.0;
  }
  __syncwarp();
  int32_t* i32 = reinterpret_cast<int32_t*>(ws) + P.n_max;  // 2 * n_max more int32
  int64_t* i64 = reinterpret_cast<int64_t*>(ws + P.i64_offset);
  switch (c.policy) {
    case BFSIM_POLICY_FCFS: fifo(w, false); break;
    case BFSIM_POLICY_JSQ: fifo(w, true); break;
    case BFSIM_POLICY_BFIO_GREEDY:
      greedy(w, i32, i32 + P.n_max, i64, i64 + 32 * (P.h_max + 1));
      break;
    case BFSIM_POLICY_BFIO_EXACT: {
      // per-lane scratch: choice, best choice (n each), loads ((H+1)*G), caps, options (n+1)
      unsigned char* lw = ws + P.lane_offset + static_cast<size_t>(lane) * P.lane_stride;
      int32_t* lchoice = reinterpret_cast<int32_t*>(lw);
      int32_t* bchoice = lchoice + P.ex_n;
      int32_t* lcap = bchoice + P.ex_n;
      int32_t* opt = lcap + 32;
      int64_t* L = reinterpret_cast<int64_t*>(lw + P.lane_i64_offset);
      exact(w, lchoice, bchoice, L, lcap, opt, P.limit, &P.cost[call], &P.status[call]);
      break;
    }
  }
  __syncwarp();
  const int64_t np = emit_pairs(w);
  if (lane == 0) P.n_pairs[call] = np;
}

}  // namespace

int launch_assign(const AssignParams& p, void* stream) {
  if (p.n_calls <= 0) return 0;
  assign_kernel<<<static_cast<unsigned>(p.n_calls), 32, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace bfsim
