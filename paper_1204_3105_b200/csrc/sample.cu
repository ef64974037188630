// sample.cu -- SURVEY §8(f) NEXT-4: device-side input generation.  Regular-polygon point
// picking in leaf cells (Fig. 12): "the polygon is subdivided into
// disjoint isosceles triangles per edge where halves of triangles are rearranged to form
// rectangles.  Uniformly random points (x,y) are picked from this rectangle and a third
// uniformly random variable z assigns the point to one of the isosceles triangles."
//
// Random numbers are counter-based (reading D22): draw d of point g is the
// SplitMix64 output h(seed, 4g + d), so a point depends only on (seed, g) -- any slice of a
// sample (a rank's cells, a sampled check) is drawn alone.  The leaf polygon comes from the
// tree's own geometry: centre by CellCenter (geometry.cuh, bit-exact form D12), the
// triangle's orientation by the parity of its centre-child digits (isUp), and
// every rounding is an explicit __d*_rn so that the points are bit-identical to the oracle's.
#include <algorithm>

#include "fmm_internal.cuh"
#include "geometry.cuh"

namespace {

__device__ __forceinline__ uint64_t smix_draw(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double unit53(uint64_t h) { return __dmul_rn((double)(h >> 11), 0x1p-53); }

// cos (k pi / 6), k = 0..20 (sin (k pi / 6) = entry k + 9; apothem directions have k <= 11)
__constant__ double SMP_COS[21] = {1.0,  FMM_H, 0.5, 0.0, -0.5, -FMM_H, -1.0, -FMM_H, -0.5, 0.0, 0.5,
                                   FMM_H, 1.0,  FMM_H, 0.5, 0.0,  -0.5,  -FMM_H, -1.0, -FMM_H, -0.5};

// one thread per point, 256-point tiles; the leaf polygons a tile touches (<= 256) are
// placed first, one per thread, in shared memory (centre, apothem-direction offset); point o
// of the call is point g = first + o of the sample
constexpr int SMP_T = 256;
__global__ void __launch_bounds__(SMP_T) k_sample_cells(DGeo g, const int64_t* __restrict__ cells, int64_t ncells,
                                                        int per_cell, uint64_t seed, int64_t first, SamplePoly P,
                                                        double2* __restrict__ xy, double* __restrict__ u,
                                                        unsigned long long* bad) {
  __shared__ double2 s_cen[SMP_T];
  __shared__ int s_off[SMP_T];
  const int64_t npts = ncells * per_cell;
  for (int64_t o0 = blockIdx.x * (int64_t)SMP_T; o0 < npts; o0 += (int64_t)gridDim.x * SMP_T) {
    const int64_t i0 = o0 / per_cell;
    const int nc = (int)((min(o0 + SMP_T, npts) - 1) / per_cell - i0 + 1);
    __syncthreads();
    if (threadIdx.x < nc) {
      const int64_t cell = cells ? cells[i0 + threadIdx.x] : i0 + threadIdx.x;
      int off = -1;
      if (cell < 0 || cell >= g.K) {
        atomicMin(bad, (unsigned long long)(i0 + threadIdx.x));
      } else {
        s_cen[threadIdx.x] = geo_centre(g, g.L, cell);
        off = P.off;
        if (g.tiling == FMM_TRIQUAD) {  // inverted (an odd number of centre-child digits): 4z + 3
          int zeros = 0;
          for (int d = 0; d < g.L; ++d) zeros += ((cell >> (2 * d)) & 3) == 0;
          off = (zeros & 1) ? 3 : 1;
        }
      }
      s_off[threadIdx.x] = off;
    }
    __syncthreads();
    const int64_t o = o0 + threadIdx.x;
    if (o >= npts) continue;
    const int q = (int)((uint32_t)(o - i0 * per_cell) / (uint32_t)per_cell);
    const int off = s_off[q];
    if (off < 0) continue;
    const double2 c = s_cen[q];
    const uint64_t gi = (uint64_t)(first + o);
    const double s = unit53(smix_draw(seed, 4 * gi)), t = unit53(smix_draw(seed, 4 * gi + 1));
    const int z = (int)(((smix_draw(seed, 4 * gi + 2) >> 32) * (uint64_t)P.nsides) >> 32);
    // rectangle a x b: s <= t is the right half of edge z's isosceles triangle, s > t its left half
    double X, Y;
    if (s > t) {
      X = __dmul_rn(__dsub_rn(s, 1.0), P.a);
      Y = __dmul_rn(__dsub_rn(1.0, t), P.b);
    } else {
      X = __dmul_rn(s, P.a);
      Y = __dmul_rn(t, P.b);
    }
    const int k = P.step * z + off;
    const double cs = SMP_COS[k], sn = SMP_COS[k + 9];  // k = step z + off <= 11
    // +Y along the apothem direction (cs, sn), +X along the edge (sn, -cs)
    const double px = __dadd_rn(__dmul_rn(Y, cs), __dmul_rn(X, sn));
    const double py = __dsub_rn(__dmul_rn(Y, sn), __dmul_rn(X, cs));
    xy[o] = make_double2(__dadd_rn(c.x, px), __dadd_rn(c.y, py));
    if (u) u[o] = __dsub_rn(__dmul_rn(2.0, unit53(smix_draw(seed, 4 * gi + 3))), 1.0);
  }
}

}  // namespace

int fmm_sample_launch(const Geo& G, const int64_t* cells, int64_t ncells, int per_cell, uint64_t seed, int64_t first,
                      const SamplePoly& P, double* xy, double* u, unsigned long long* bad, cudaStream_t s) {
  const int64_t npts = ncells * per_cell;
  if (npts > 0) {
    const int64_t blocks = std::min<int64_t>((npts + SMP_T - 1) / SMP_T, 148 * 8 * 16);
    k_sample_cells<<<(unsigned)blocks, SMP_T, 0, s>>>(dgeo(G), cells, ncells, per_cell, seed, first, P, (double2*)xy,
                                                    u, bad);
  }
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}
