// Leaf-binned query pipeline (capt_binned.cu) -- shared declarations.
#pragma once

#include "capt_internal.cuh"

namespace capt {

// One K5 work item: up to 1024 binned spheres of one leaf, with everything
// K5 needs to start it (one 48-B load instead of a chain of dependent ones).
struct __align__(16) TileMeta {
  int leaf;
  uint32_t s0;    // first binned slot
  int cnt;        // spheres in the tile
  uint32_t setx;  // set start (float4 units)
  uint32_t m;     // set size
  uint32_t pad[3];
  float4 org;     // binned-scan origin of the set
};

struct BinArgs {
  DevTree t;
  const void* centers;
  const void* radii;
  int64_t n;
  int L;
  const uint8_t* mask;
  uint32_t flags;
  uint32_t* counts;   // per leaf: AABB-passing spheres
  uint32_t* start;    // per leaf: first binned slot
  uint32_t* tstart;   // per order index: first tile
  TileMeta* tiles;
  uint8_t* verdict;   // per sphere
  int2* slow;         // (sphere, leaf) for the exact float64 path
  uint32_t* slow_n;
  uint32_t* n_tiles;
  uint32_t* tile_ctr;
  uint32_t* n_refined;
  unsigned long long* first_bad;
  float4* lrec;       // compact list of binned spheres (K1 -> K3): {c, r}
  int2* lmeta;        //   ... and (sphere id, leaf)
  uint8_t* lhit;      //   ... and K5's hit flag (mapped back to spheres by K6)
  uint32_t* list_n;   //   ... length
  uint32_t* cursor;   // per leaf: scatter cursor (K3b)
  int2* part;         // K3a output: (leaf, list index), grouped by leaf bucket
  uint32_t* perm;     // K3b output: list index of binned slot i (leaf order)
  uint32_t* bcursor;  // per leaf bucket: K3a cursor
  int bshift;         // leaf bucket = leaf >> bshift (<= kBuckets buckets)
  float rlo_f, rhi_f; // fp32 images of the double band edges
  uint32_t ts;        // spheres per K5 tile (kernel dependent)
};

bool binned_preferred(const DevTree& t, int64_t n, uint32_t flags);

int launch_binned(const DevTree& t, const void* centers, const void* radii, int64_t n, int L,
                  const uint8_t* mask, uint32_t flags, uint32_t* bits, int64_t n_words,
                  unsigned long long* first_bad, cudaStream_t s);

}  // namespace capt
