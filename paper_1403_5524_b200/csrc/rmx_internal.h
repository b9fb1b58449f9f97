// rmx_internal.h - launcher declarations shared by the librmx translation units (not installed).
#pragma once
#include <cstdint>
#include <string>
#include <cuda_runtime.h>
#include "../../include/rmx.h"

namespace rmx {

// rform.cu
int rform_tile_for(int64_t nch);
cudaError_t launch_rform(const double *w, int64_t ldw, const double *Ek, int64_t nch, int64_t nlev,
                         double a, const double *E, int64_t ne, double *R, int32_t *status,
                         cudaStream_t st, std::string &err);

// match.cu
size_t match_smem_bytes();
int64_t match_ws_doubles_per_slot(int64_t nch);
cudaError_t launch_match(const double *R, const double *F, const double *G, const double *Fp,
                         const double *Gp, double a, int64_t nch, int64_t ne, const int32_t *n_open,
                         double *K, double *ws, int64_t ws_slots, int32_t *status, cudaStream_t st);

// tepi.cu
int64_t tepi_ws_doubles_per_slot(int64_t nch);
cudaError_t launch_tepi(const double *K, int64_t ldk, int64_t kstride, int64_t nch, int64_t ne,
                        const int32_t *n_open, double *T2, const int64_t *t2_slot, double *rowsum,
                        double *ws, int64_t ws_slots, int32_t *status, cudaStream_t st);

}  // namespace rmx
