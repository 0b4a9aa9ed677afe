// wm_dict.cu — the pattern dictionary (reference build_dictionary,
// pkg/src/warpmine/canon.py:315-343) built on the device.
//
// The reference scans every reachable bitmap in ascending order in Python;
// the first unseen member of an isomorphism class is the class minimum, and
// one vectorised pass over the k! relabelings fills the whole orbit
// (canon.py:22-26).  At k = 8 that scan walks ~1e8 Python ints and is
// impractical (the CLI gates it behind --allow-large, cli.py:71-72).  Here the
// same sweep runs on the GPU:
//   find_next_kernel  one block scans the table forward from a device cursor
//                     for the first reachable bitmap still SENTINEL (the next
//                     class minimum), assigns it the next pattern id;
//   orbit_kernel      one thread per relabeling applies the permutation's
//                     slot map to that bitmap and writes the id for every
//                     valid image (canon.py:118-167 semantics).
// Pairs of launches are queued in batches without host round trips; the
// class order, ids and table bytes are exactly the reference's.
#include "wm_common.cuh"

#include <algorithm>
#include <vector>

namespace wm {

namespace {

constexpr uint32_t kSentinel = 0xFFFFFFFFu;

struct DictArgs {
  uint32_t *table;
  unsigned long long size;       // 2^nbits
  int k, nbits;
  const uint8_t *slots;          // [nperm][nbits + 1] destination full-slot index
  int nperm;
  unsigned long long *cursor;    // next bitmap to examine
  unsigned long long *current;   // class minimum found by the last find
  uint32_t *count;               // pattern ids assigned
  unsigned long long *bitmaps;   // [cap] canonical bitmaps
  uint32_t cap;
  int *done;
};

__device__ __forceinline__ bool reachable(unsigned long long v, int k) {
  // every vertex group i >= 2 non-zero (canon.py:107-112)
  for (int i = 2; i < k; ++i) {
    const int off = i * (i - 1) / 2 - 1;
    if (((v >> off) & ((1ull << i) - 1ull)) == 0ull) return false;
  }
  return true;
}

__global__ void __launch_bounds__(1024) find_next_kernel(DictArgs a) {
  __shared__ unsigned long long best;
  if (*a.done) return;
  const unsigned long long W = 1ull << 16;
  for (unsigned long long base = *a.cursor; base < a.size; base += W) {
    if (threadIdx.x == 0) best = ~0ull;
    __syncthreads();
    unsigned long long mine = ~0ull;
    for (unsigned long long v = base + threadIdx.x; v < base + W && v < a.size; v += blockDim.x) {
      if (reachable(v, a.k) && a.table[v] == kSentinel) { mine = v; break; }
    }
    if (mine != ~0ull) atomicMin(&best, mine);
    __syncthreads();
    const unsigned long long b = best;
    __syncthreads();
    if (b != ~0ull) {
      if (threadIdx.x == 0) {
        const uint32_t pid = *a.count;
        if (pid < a.cap) a.bitmaps[pid] = b;
        *a.count = pid + 1;
        *a.current = b;
        *a.cursor = b + 1;
      }
      return;
    }
  }
  if (threadIdx.x == 0) *a.done = 1;
}

__global__ void __launch_bounds__(256) orbit_kernel(DictArgs a) {
  if (*a.done) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.nperm) return;
  const unsigned long long b = *a.current;
  const uint32_t pid = *a.count - 1;
  const int nb = a.nbits;
  const unsigned long long full = b | (1ull << nb);  // implicit (v1, v0) edge on the top slot
  const uint8_t *dst = a.slots + (size_t)p * (nb + 1);
  unsigned long long img = 0;
  for (int sl = 0; sl <= nb; ++sl)
    if ((full >> sl) & 1ull) img |= 1ull << dst[sl];
  // valid image: top slot set and every stored group non-zero (canon.py:150-155)
  if (!((img >> nb) & 1ull)) return;
  const unsigned long long stored = img & ((1ull << nb) - 1ull);
  if (!reachable(stored, a.k)) return;
  a.table[stored] = pid;
}

int stored_bits_of(int k) { return k * (k - 1) / 2 - 1; }

int full_slot(int i, int j, int nbits) { return i == 1 ? nbits : i * (i - 1) / 2 - 1 + j; }

}  // namespace

}  // namespace wm

using namespace wm;

extern "C" int wm_dictionary_build(int k, uint32_t *table_out, uint64_t *bitmaps_out,
                                   uint32_t bitmaps_cap, uint32_t *pattern_count) {
  clear_error();
  if (k < 3 || k > 8) return fail(WM_EINVAL, "dictionary supports 3 <= k <= 8, got k=%d", k);
  if (!table_out || !pattern_count) return fail(WM_EINVAL, "null argument");
  Workspace *ws = nullptr;
  int st = workspace_get(&ws);
  if (st) return st;
  WsLock lk(ws);
  if ((st = lk.status())) return st;
  cudaStream_t s = ws->own_stream;
  const int nbits = stored_bits_of(k);
  const unsigned long long size = 1ull << nbits;
  // relabeling slot maps (canon.py:118-139)
  std::vector<int> perm(k);
  for (int i = 0; i < k; ++i) perm[i] = i;
  std::vector<uint8_t> slots;
  int nperm = 0;
  do {
    std::vector<uint8_t> row(nbits + 1);
    for (int i = 1; i < k; ++i)
      for (int j = 0; j < i; ++j) {
        int a = perm[i], b = perm[j];
        if (a < b) std::swap(a, b);
        row[full_slot(i, j, nbits)] = (uint8_t)full_slot(a, b, nbits);
      }
    slots.insert(slots.end(), row.begin(), row.end());
    ++nperm;
  } while (std::next_permutation(perm.begin(), perm.end()));
  DeviceBuffer dtable, dslots, dstate, dbitmaps;
  if ((st = dtable.ensure(sizeof(uint32_t) * size))) return st;
  if ((st = dslots.ensure(slots.size()))) return st;
  if ((st = dstate.ensure(64))) return st;
  const uint32_t cap = bitmaps_cap > 0 ? bitmaps_cap : 1;
  if ((st = dbitmaps.ensure(sizeof(unsigned long long) * cap))) return st;
  WM_CUDA(cudaMemsetAsync(dtable.ptr, 0xff, sizeof(uint32_t) * size, s));
  WM_CUDA(cudaMemsetAsync(dstate.ptr, 0, 64, s));
  WM_CUDA(cudaMemcpyAsync(dslots.ptr, slots.data(), slots.size(), cudaMemcpyHostToDevice, s));
  DictArgs a;
  a.table = dtable.as<uint32_t>();
  a.size = size;
  a.k = k;
  a.nbits = nbits;
  a.slots = dslots.as<uint8_t>();
  a.nperm = nperm;
  char *base = dstate.as<char>();
  a.cursor = reinterpret_cast<unsigned long long *>(base);
  a.current = reinterpret_cast<unsigned long long *>(base + 8);
  a.count = reinterpret_cast<uint32_t *>(base + 16);
  a.done = reinterpret_cast<int *>(base + 20);
  a.bitmaps = dbitmaps.as<unsigned long long>();
  a.cap = cap;
  const int oblocks = (nperm + 255) / 256;
  int done = 0;
  while (!done) {
    for (int it = 0; it < 256; ++it) {
      find_next_kernel<<<1, 1024, 0, s>>>(a);
      orbit_kernel<<<oblocks, 256, 0, s>>>(a);
    }
    WM_CUDA(cudaGetLastError());
    WM_CUDA(cudaMemcpyAsync(&done, a.done, sizeof done, cudaMemcpyDeviceToHost, s));
    WM_CUDA(cudaStreamSynchronize(s));
  }
  uint32_t count = 0;
  WM_CUDA(cudaMemcpyAsync(&count, a.count, sizeof count, cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  *pattern_count = count;
  if (count > bitmaps_cap)
    return fail(WM_ECAPACITY, "%u patterns exceed the bitmap buffer (%u)", count, bitmaps_cap);
  WM_CUDA(cudaMemcpyAsync(table_out, dtable.ptr, sizeof(uint32_t) * size, cudaMemcpyDeviceToHost,
                          s));
  if (bitmaps_out && count)
    WM_CUDA(cudaMemcpyAsync(bitmaps_out, dbitmaps.ptr, sizeof(unsigned long long) * count,
                            cudaMemcpyDeviceToHost, s));
  WM_CUDA(cudaStreamSynchronize(s));
  return WM_OK;
}
