// gc_band.cpp — row-band domain decomposition over NCCL.
//
// Each rank owns contiguous rows of one large image.  Eq. (7) at row y reads rows
// y-W_s .. y+W_s, and the N+2 auxiliary planes of eq. (6) are pointwise in f, so the
// only data a band needs from its neighbours are W_s rows of f above and below.  They
// are exchanged with one grouped ncclSend/ncclRecv per neighbour (NVLink/NVSwitch on
// one node), then the band is filtered by gc_filter_window with three input segments
// (top halo, own band, bottom halo).  Symmetric extension is applied only at the
// global rows 0 and H-1, so the result equals the single-GPU filter of the whole image.
#include <cmath>
#include <cstring>
#include <vector>

#include <nccl.h>

#include "gc_internal.h"

extern "C" {

gc_status gc_band_plan(int H_global, int rank, int world, const int* band_rows, float sigma_s, int* row0,
                       int* top0, int* top_rows, int* bot0, int* bot_rows) {
  if (!band_rows || world < 1 || rank < 0 || rank >= world || H_global < 1) return GC_EINVAL;
  if (!(std::isfinite(sigma_s) && sigma_s > 0)) return GC_EINVAL;
  const int R = (int)std::ceil(3.0 * (double)sigma_s);
  long long sum = 0, r0 = 0;
  for (int k = 0; k < world; k++) {
    if (band_rows[k] < 1) return GC_EINVAL;
    if (world > 1 && band_rows[k] <= R) return GC_EINVAL;   // halos from adjacent ranks only
    if (k < rank) r0 += band_rows[k];
    sum += band_rows[k];
  }
  if (sum != H_global) return GC_EINVAL;
  const int hb = band_rows[rank];
  if (row0) *row0 = (int)r0;
  if (top0) *top0 = (int)r0 - (rank > 0 ? R : 0);
  if (top_rows) *top_rows = rank > 0 ? R : 0;
  if (bot0) *bot0 = (int)r0 + hb;
  if (bot_rows) *bot_rows = rank < world - 1 ? R : 0;
  return GC_OK;
}

gc_status gc_comm_unique_id(unsigned char id[128]) {
  if (!id) return GC_EINVAL;
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return GC_ENCCL;
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return GC_OK;
}

gc_status gc_comm_init(int rank, int world, const unsigned char id[128], void** comm_out) {
  if (!id || !comm_out || world < 1 || rank < 0 || rank >= world) return GC_EINVAL;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c;
  if (ncclCommInitRank(&c, world, u, rank) != ncclSuccess) return GC_ENCCL;
  *comm_out = c;
  return GC_OK;
}

gc_status gc_comm_destroy(void* comm) {
  if (!comm) return GC_EINVAL;
  return ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm)) == ncclSuccess ? GC_OK : GC_ENCCL;
}

gc_status gc_bilateral_band(const float* band, int H_band, int W, int H_global, int row0, const gc_params* p,
                            float* out, void* comm, void* stream) {
  if (!band || !out || !comm || !p || H_band < 1 || W < 1 || row0 < 0 || row0 + H_band > H_global)
    return GC_EINVAL;
  if (!(std::isfinite(p->sigma_s) && p->sigma_s > 0)) return GC_EINVAL;
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
  int rank = 0, world = 1;
  if (ncclCommUserRank(c, &rank) != ncclSuccess || ncclCommCount(c, &world) != ncclSuccess) return GC_ENCCL;
  // halo rows: W_s for eq. (7); the Deriche operator's lead-in K = ceil(10 sigma_s) for GC_OP_DERICHE
  const int R = (int)std::ceil((p->op == GC_OP_DERICHE ? 10.0 : 3.0) * (double)p->sigma_s);
  const bool has_top = rank > 0, has_bot = rank < world - 1;
  if ((has_top || has_bot) && H_band <= R) return GC_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t halo = (size_t)R * W;
  float *top = nullptr, *bot = nullptr;
  if (has_top && cudaMallocAsync((void**)&top, halo * 4, s) != cudaSuccess) return GC_ENOMEM;
  if (has_bot && cudaMallocAsync((void**)&bot, halo * 4, s) != cudaSuccess) {
    if (top) cudaFreeAsync(top, s);
    return GC_ENOMEM;
  }
  gc_status st = GC_OK;
  if (ncclGroupStart() != ncclSuccess) st = GC_ENCCL;
  if (st == GC_OK && has_top) {
    // my first R rows go up; the R rows above me come down from rank-1
    if (ncclSend(band, halo, ncclFloat32, rank - 1, c, s) != ncclSuccess) st = GC_ENCCL;
    if (ncclRecv(top, halo, ncclFloat32, rank - 1, c, s) != ncclSuccess) st = GC_ENCCL;
  }
  if (st == GC_OK && has_bot) {
    if (ncclSend(band + (size_t)(H_band - R) * W, halo, ncclFloat32, rank + 1, c, s) != ncclSuccess) st = GC_ENCCL;
    if (ncclRecv(bot, halo, ncclFloat32, rank + 1, c, s) != ncclSuccess) st = GC_ENCCL;
  }
  if (ncclGroupEnd() != ncclSuccess) st = GC_ENCCL;
  if (st == GC_OK) {
    const float* seg[3] = {has_top ? top : band, band, has_bot ? bot : band};
    const int seg_row0[3] = {row0 - R, row0, row0 + H_band};
    const int seg_rows[3] = {has_top ? R : 0, H_band, has_bot ? R : 0};
    st = gc_filter_window(seg, seg_row0, seg_rows, H_global, W, row0, H_band, p, out, stream);
  }
  if (top) cudaFreeAsync(top, s);
  if (bot) cudaFreeAsync(bot, s);
  return st;
}

}  // extern "C"
