// Internal launcher declarations (not part of the public ABI).
#pragma once
#include "lf_b200.h"
#include "lf_common.cuh"

int lf_launch_ewise(const LfCtx* ctx, int op, u32* out, const u32* a, const u32* b,
                    const u32* c, const RowMap& rm, const u32* scalars, cudaStream_t s);
int lf_launch_automorph(const LfCtx* ctx, u32* out, const u32* in, u32 g, int nrows,
                        cudaStream_t s);
int lf_launch_bconv(const LfCtx* ctx, u32* out, const u32* src, const u32* tab, int k, int m,
                    int W, cudaStream_t s);

#define LF_PTMAC_MAX 32
int lf_launch_modraise(const LfCtx* ctx, u32* out, const u32* in, int nin, int nout,
                       cudaStream_t s);
int lf_launch_ptmac(const LfCtx* ctx, u32* out, int nrows, int nterm, const u32* const* b,
                    const u32* const* a, const u32* const* pt, const int32_t* pidx, cudaStream_t s);
#define LF_LINCOMB_MAX 8
#define LF_LINCOMB_ROWS 64
int lf_launch_lincomb(const LfCtx* ctx, u32* out, int nrows, int nterm, const u32* const* b,
                      const u32* const* a, const u32* k, const u32* cb, cudaStream_t s);
int lf_launch_convert(void* out, const void* in, size_t n, bool narrow, cudaStream_t s);
int lf_launch_mul_compressed(const LfCtx* ctx, u32* out, const u32* ct, const u32* uq, int nrows,
                             int ucount, int lb, cudaStream_t s);
int lf_launch_plan_step(const LfCtx* ctx, const void* ops, int nops, cudaStream_t s);
