// Full-space StVK implicit Euler on the GPU (elastic.fullspace_step, SPEC.md:344-352;
// SURVEY.md §8f rank 2): ground truth for the reduced trajectories and the integrator of the
// pose generator (posegen.generate_poses).
//
// Per step, Newton on v':
//   g(v') = M (v' - v) / dt + (alpha M + beta K(u')) v' + f_int(u') - f_ext,  u' = u + dt v'
//   [(1 + alpha dt) M + (beta dt + dt^2) K(u')] dv = -dt g        (dK/du v' dropped)
// Kernels (one stream, deterministic -- every sum has a fixed order):
//   k_fs_elements   warp per tet: F, Green strain, S, P (StVK), f_e (12),
//                   K_e (12 x 12, lane = column), volume-weighted energy; block energy partials
//   k_fs_assemble   thread per CSR nonzero: K_ij = sum of its K_e entries (precomputed
//                   contribution lists in element order), H_ij = c_K K_ij + c_M M_i delta_ij
//   k_fs_residual   thread per DOF: f_int by row gather (no atomics), scaled residual
//                   dt g, Jacobi diagonal, block partials of ||g||^2
//   k_fs_pcg        ONE cooperative kernel for the whole Jacobi-PCG solve: warp-per-row SpMV
//                   (L2-resident CSR), grid-wide syncs between the phases, every dot product
//                   as fixed-order block partials that every block re-sums identically
// The CSR pattern, the assembly lists and the force gather lists are built once on the host.
#include <cooperative_groups.h>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>
#include "common.cuh"

namespace cg = cooperative_groups;

namespace nlrom {

struct FsElemArgs {
  const int* rows;      // (T,12) free-DOF rows, -1 fixed
  const double* Dm_inv; // (T,9)
  const double* vol;    // (T,)
  const double* u;      // (N,)
  int T;
  double mu, lam;
  double* fe;           // (T,12)
  double* Ke;           // (T,144) row-major K_e[r][c] (nullable)
  double* epart;        // (gridDim.x,) energy partials
};

__device__ __forceinline__ void fs_mat3(const double* A, const double* B, double* C) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) C[i * 3 + j] = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
}

__global__ void __launch_bounds__(256) k_fs_elements(FsElemArgs a) {
  __shared__ double es[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * 8 + warp;
  double energy = 0.0;
  if (e < a.T) {
    double ue = 0.0;
    if (lane < 12) {
      const int row = a.rows[(size_t)e * 12 + lane];
      ue = row >= 0 ? a.u[row] : 0.0;
    }
    double uv[12];
#pragma unroll
    for (int l = 0; l < 12; ++l) uv[l] = __shfl_sync(0xffffffffu, ue, l);
    double Di[9];
#pragma unroll
    for (int l = 0; l < 9; ++l) Di[l] = a.Dm_inv[(size_t)e * 9 + l];
    const double V = a.vol[e];
    // gradient rows g_i (i = 1..3: rows of Dm^-1; g_0 = -sum)
    double G[12];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      G[3 + b] = Di[b];
      G[6 + b] = Di[3 + b];
      G[9 + b] = Di[6 + b];
      G[b] = -(Di[b] + Di[3 + b] + Di[6 + b]);
    }
    double Ds[9], F[9];
#pragma unroll
    for (int aa = 0; aa < 3; ++aa)
#pragma unroll
      for (int i = 0; i < 3; ++i) Ds[aa * 3 + i] = uv[(i + 1) * 3 + aa] - uv[aa];
    fs_mat3(Ds, Di, F);
    F[0] += 1.0;
    F[4] += 1.0;
    F[8] += 1.0;
    double E[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        E[i * 3 + j] = 0.5 * (F[i] * F[j] + F[3 + i] * F[3 + j] + F[6 + i] * F[6 + j] - (i == j ? 1.0 : 0.0));
    const double trE = E[0] + E[4] + E[8];
    if (lane == 0) {
      double ee = 0.0;
#pragma unroll
      for (int l = 0; l < 9; ++l) ee = fma(E[l], E[l], ee);
      energy = V * (a.mu * ee + 0.5 * a.lam * trE * trE);
    }
    double S[9];
#pragma unroll
    for (int l = 0; l < 9; ++l) S[l] = 2.0 * a.mu * E[l];
    S[0] += a.lam * trE;
    S[4] += a.lam * trE;
    S[8] += a.lam * trE;
    double P[9];
    fs_mat3(F, S, P);
    if (lane < 12) {
      const int i = lane / 3, aa = lane % 3;
      a.fe[(size_t)e * 12 + lane] =
          V * (P[aa * 3] * G[i * 3] + P[aa * 3 + 1] * G[i * 3 + 1] + P[aa * 3 + 2] * G[i * 3 + 2]);
      if (a.Ke) {
        // stiffness column for DOF (jv, d) = lane: dF_ab = delta_ad g_jv[b]
        const int jv = lane / 3, d = lane % 3;
        double dF[9];
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int y = 0; y < 3; ++y) dF[x * 3 + y] = (x == d) ? G[jv * 3 + y] : 0.0;
        double dE[9];
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int y = 0; y < 3; ++y)
            dE[x * 3 + y] = 0.5 * (dF[x] * F[y] + dF[3 + x] * F[3 + y] + dF[6 + x] * F[6 + y] + F[x] * dF[y] +
                                   F[3 + x] * dF[3 + y] + F[6 + x] * dF[6 + y]);
        const double trdE = dE[0] + dE[4] + dE[8];
        double dS[9];
#pragma unroll
        for (int l = 0; l < 9; ++l) dS[l] = 2.0 * a.mu * dE[l];
        dS[0] += a.lam * trdE;
        dS[4] += a.lam * trdE;
        dS[8] += a.lam * trdE;
        double t1[9], t2[9];
        fs_mat3(dF, S, t1);
        fs_mat3(F, dS, t2);
#pragma unroll
        for (int l = 0; l < 9; ++l) t1[l] += t2[l];
#pragma unroll
        for (int r = 0; r < 12; ++r) {
          const int ri = r / 3, ra = r % 3;
          a.Ke[(size_t)e * 144 + r * 12 + lane] =
              V * (t1[ra * 3] * G[ri * 3] + t1[ra * 3 + 1] * G[ri * 3 + 1] + t1[ra * 3 + 2] * G[ri * 3 + 2]);
        }
      }
    }
  }
  if (lane == 0) es[warp] = energy;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += es[w];
    a.epart[blockIdx.x] = s;
  }
}

// K (and H = cK K + cM M) on the CSR pattern; contributions summed in element order
__global__ void k_fs_assemble(const int* __restrict__ aptr, const int* __restrict__ alist, const int* __restrict__ nz_row,
                              const unsigned char* __restrict__ is_diag, const double* __restrict__ Ke,
                              const double* __restrict__ mass, double cK, double cM, int nnz, double* __restrict__ Kv,
                              double* __restrict__ Hv) {
  for (int z = blockIdx.x * blockDim.x + threadIdx.x; z < nnz; z += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = aptr[z]; t < aptr[z + 1]; ++t) s += Ke[alist[t]];
    Kv[z] = s;
    Hv[z] = cK * s + (is_diag[z] ? cM * mass[nz_row[z]] : 0.0);
  }
}

// scaled residual rs = dt g, b = -rs, Jacobi diagonal, block partials of ||g||^2
__global__ void __launch_bounds__(256) k_fs_residual(const int* __restrict__ fptr, const int* __restrict__ flist,
                                                     const double* __restrict__ fe, const int* __restrict__ rp,
                                                     const int* __restrict__ col, const double* __restrict__ Kv,
                                                     const double* __restrict__ Hv, const int* __restrict__ dpos,
                                                     const double* __restrict__ mass, const double* __restrict__ x,
                                                     const double* __restrict__ v, const double* __restrict__ fext,
                                                     double dt, double alpha, double beta, int N,
                                                     double* __restrict__ b, double* __restrict__ dinv,
                                                     double* __restrict__ fint, double* __restrict__ gpart) {
  __shared__ double red[8];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double g2 = 0.0;
  if (i < N) {
    double f = 0.0;
    for (int t = fptr[i]; t < fptr[i + 1]; ++t) f += fe[flist[t]];
    fint[i] = f;
    double kx = 0.0;
    if (beta != 0.0)
      for (int k = rp[i]; k < rp[i + 1]; ++k) kx = fma(Kv[k], x[col[k]], kx);
    const double m = mass[i];
    const double g = m * (x[i] - v[i]) / dt + alpha * m * x[i] + beta * kx + f - fext[i];
    b[i] = -dt * g;
    dinv[i] = 1.0 / Hv[dpos[i]];
    g2 = g * g;
  }
  for (int o = 16; o; o >>= 1) g2 += __shfl_down_sync(0xffffffffu, g2, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = g2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    gpart[blockIdx.x] = s;
  }
}

__global__ void k_fs_axpy(double* __restrict__ y, const double* __restrict__ base, const double* __restrict__ d,
                          double t, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = base[i] + t * d[i];
}

// ------------------------------------------------------------------ cooperative Jacobi-PCG
struct PcgArgs {
  const int* rp;
  const int* col;
  const double* A;
  const double* dinv;
  const double* b;
  double* x;
  double* r;
  double* z;
  double* p;
  double* Ap;
  double* part;   // (gridDim.x, 4)
  int N;
  double tol;
  int maxit;
  int* iters;
  double* relres;
};

constexpr int PCG_NTH = 1024;  // 32 warps per block: rows of the latency-bound SpMV in flight
constexpr int PCG_NW = PCG_NTH / 32;

// block-wide sum, fixed order; result in every thread
__device__ __forceinline__ double pcg_block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < PCG_NW; ++w) s += red[w];
  return s;
}

// sum of the blocks' partials (slot k) in a fixed order, identical in every block
__device__ __forceinline__ double pcg_grid_sum(const double* part, int k, int nb, double* red) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  if (threadIdx.x < 32)
    for (int i = lane; i < nb; i += 32) v += __ldcg(part + (size_t)i * 4 + k);
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if (threadIdx.x == 0) red[PCG_NW] = v;
  __syncthreads();
  return red[PCG_NW];
}

// Two grid-wide syncs per iteration: the direction update p = z + beta p_prev is not a phase of
// its own -- the SpMV forms it on the fly for every column it reads (the owner block stores it
// for its rows in the other buffer of p), with exactly the same expression, so all blocks see
// the same p bits.
__device__ __forceinline__ double pcg_dir(double z, double beta, double pprev) { return fma(beta, pprev, z); }

__global__ void __launch_bounds__(PCG_NTH) k_fs_pcg(PcgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[PCG_NW + 1];
  const int nb = gridDim.x, blk = blockIdx.x, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int per = (a.N + nb - 1) / nb;
  const int r0 = min(a.N, blk * per), r1 = min(a.N, r0 + per);
  double* P[2] = {a.p, a.Ap + a.N};  // direction buffers (Ap has room for 2N)
  double lrz = 0.0, lbb = 0.0;
  for (int i = r0 + tid; i < r1; i += blockDim.x) {
    const double bi = a.b[i], zi = a.dinv[i] * bi;
    a.x[i] = 0.0;
    a.r[i] = bi;
    a.z[i] = zi;
    P[1][i] = 0.0;  // p_prev of iteration 0 (beta = 0)
    lrz += bi * zi;
    lbb += bi * bi;
  }
  lrz = pcg_block_sum(lrz, red);
  lbb = pcg_block_sum(lbb, red);
  if (tid == 0) {
    a.part[blk * 4 + 0] = lrz;
    a.part[blk * 4 + 1] = lbb;
  }
  grid.sync();
  double rz = pcg_grid_sum(a.part, 0, nb, red);
  const double bb = pcg_grid_sum(a.part, 1, nb, red);
  const double thr = a.tol * a.tol * bb;
  double rr = bb, beta = 0.0;
  int it = 0;
  while (bb > 0.0 && it < a.maxit) {
    double* pc = P[it & 1];
    const double* pp = P[(it + 1) & 1];
    // Ap = A p with p = z + beta p_prev formed per column read (warp per row), partial p . Ap
    double lpap = 0.0;
    for (int i = r0 + warp; i < r1; i += PCG_NW) {
      double s = 0.0;
      for (int k = a.rp[i] + lane; k < a.rp[i + 1]; k += 32) {
        const int c = a.col[k];
        s = fma(a.A[k], pcg_dir(__ldcg(a.z + c), beta, __ldcg(pp + c)), s);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        const double pi = pcg_dir(__ldcg(a.z + i), beta, __ldcg(pp + i));
        pc[i] = pi;
        a.Ap[i] = s;
        lpap += pi * s;
      }
    }
    lpap = pcg_block_sum(lpap, red);
    if (tid == 0) a.part[blk * 4 + 2] = lpap;
    grid.sync();
    const double pap = pcg_grid_sum(a.part, 2, nb, red);
    const double alpha = rz / pap;
    double lrz2 = 0.0, lrr = 0.0;
    for (int i = r0 + tid; i < r1; i += blockDim.x) {
      a.x[i] += alpha * __ldcg(pc + i);
      const double ri = a.r[i] - alpha * __ldcg(a.Ap + i);
      a.r[i] = ri;
      const double zi = a.dinv[i] * ri;
      a.z[i] = zi;
      lrz2 += ri * zi;
      lrr += ri * ri;
    }
    lrz2 = pcg_block_sum(lrz2, red);
    lrr = pcg_block_sum(lrr, red);
    if (tid == 0) {
      a.part[blk * 4 + 0] = lrz2;
      a.part[blk * 4 + 1] = lrr;
    }
    grid.sync();
    const double rz2 = pcg_grid_sum(a.part, 0, nb, red);
    rr = pcg_grid_sum(a.part, 1, nb, red);
    ++it;
    if (!(rr > thr)) break;  // converged (or NaN: stop, the host sees it)
    beta = rz2 / rz;
    rz = rz2;
  }
  if (blk == 0 && tid == 0) {
    *a.iters = it;
    *a.relres = bb > 0.0 ? sqrt(rr / bb) : 0.0;
  }
}

}  // namespace nlrom

using namespace nlrom;

struct nlrom_fs {
  int device = 0;
  std::string err;
  cudaStream_t st = nullptr;
  int N = 0, T = 0, nnz = 0;
  double alpha = 0, beta = 0, mu = 0, lam = 0;
  IBuf rows, rp, col, aptr, alist, nzrow, fptr, flist, dpos, iters;
  DBuf Dm_inv, vol, mass, u, v, x, up, fext, fe, Ke, epart, Kv, Hv, b, dinv, fint, gpart;
  DBuf cg_x, cg_r, cg_z, cg_p, cg_Ap, cg_part, relres;
  unsigned char* isdiag = nullptr;
  int pcg_blocks = 0;
  std::vector<double> hpart;
};

static int fs_fail(nlrom_fs* f, const Error& e) {
  f->err = e.what();
  return e.code;
}

#define FS_TRY(f)                    \
  if (!(f)) return NLROM_ERR_ARG;    \
  try {                              \
    NL_CUDA(cudaSetDevice((f)->device));
#define FS_END(f)            \
  return NLROM_OK;           \
  }                          \
  catch (const Error& e) {   \
    return fs_fail((f), e);  \
  }

extern "C" const char* nlrom_fs_last_error(const nlrom_fs* f) { return f ? f->err.c_str() : "null handle"; }

extern "C" void nlrom_fs_destroy(nlrom_fs* f) {
  if (!f) return;
  cudaSetDevice(f->device);
  if (f->isdiag) cudaFree(f->isdiag);
  if (f->st) cudaStreamDestroy(f->st);
  delete f;
}

extern "C" int nlrom_fs_create(nlrom_fs** out, int device, const nlrom_fs_desc* d) {
  if (!out || !d) return NLROM_ERR_ARG;
  *out = nullptr;
  nlrom_fs* f = new nlrom_fs();
  f->device = device;
  try {
    NL_CUDA(cudaSetDevice(device));
    NL_CUDA(cudaStreamCreateWithFlags(&f->st, cudaStreamNonBlocking));
    const int V = d->n_verts, T = d->n_tets;
    if (V <= 0 || T <= 0) throw Error(NLROM_ERR_ARG, "empty mesh");
    int nfree = 0;
    for (int i = 0; i < V; ++i) nfree = std::max(nfree, d->vert_dof[i] + 1);
    const int N = 3 * nfree;
    if (N <= 0) throw Error(NLROM_ERR_ARG, "no free DOFs");
    f->N = N;
    f->T = T;
    f->alpha = d->alpha;
    f->beta = d->beta;
    f->mu = d->mu;
    f->lam = d->lambda;
    // element rows
    std::vector<int> rows((size_t)T * 12);
    for (int e = 0; e < T; ++e)
      for (int k = 0; k < 4; ++k) {
        const int vtx = d->tets[(size_t)e * 4 + k];
        if (vtx < 0 || vtx >= V) throw Error(NLROM_ERR_ARG, "tet index out of range");
        const int fd = d->vert_dof[vtx];
        for (int c = 0; c < 3; ++c) rows[(size_t)e * 12 + 3 * k + c] = fd >= 0 ? 3 * fd + c : -1;
      }
    // CSR pattern: free-vertex adjacency expanded to 3 x 3 blocks
    std::vector<std::vector<int>> adj(nfree);
    for (int e = 0; e < T; ++e)
      for (int a = 0; a < 4; ++a) {
        const int va = d->vert_dof[d->tets[(size_t)e * 4 + a]];
        if (va < 0) continue;
        for (int b2 = 0; b2 < 4; ++b2) {
          const int vb = d->vert_dof[d->tets[(size_t)e * 4 + b2]];
          if (vb >= 0) adj[va].push_back(vb);
        }
      }
    for (auto& l : adj) {
      std::sort(l.begin(), l.end());
      l.erase(std::unique(l.begin(), l.end()), l.end());
    }
    std::vector<int> rp(N + 1, 0), col;
    for (int i = 0; i < N; ++i) {
      for (int vb : adj[i / 3])
        for (int c = 0; c < 3; ++c) col.push_back(3 * vb + c);
      rp[i + 1] = (int)col.size();
    }
    const int nnz = (int)col.size();
    f->nnz = nnz;
    std::vector<int> dpos(N), nzrow(nnz);
    std::vector<unsigned char> isd(nnz, 0);
    for (int i = 0; i < N; ++i)
      for (int k = rp[i]; k < rp[i + 1]; ++k) {
        nzrow[k] = i;
        if (col[k] == i) {
          dpos[i] = k;
          isd[k] = 1;
        }
      }
    auto find_nz = [&](int i, int j) {
      const int* b0 = col.data() + rp[i];
      const int* b1 = col.data() + rp[i + 1];
      const int* p = std::lower_bound(b0, b1, j);
      if (p == b1 || *p != j) throw Error(NLROM_ERR_ARG, "internal: CSR pattern");
      return (int)(p - col.data());
    };
    // assembly lists (element order) and force gather lists
    std::vector<int> acnt(nnz + 1, 0), fcnt(N + 1, 0);
    for (int e = 0; e < T; ++e)
      for (int li = 0; li < 12; ++li) {
        const int ri = rows[(size_t)e * 12 + li];
        if (ri < 0) continue;
        ++fcnt[ri + 1];
        for (int lj = 0; lj < 12; ++lj) {
          const int cj = rows[(size_t)e * 12 + lj];
          if (cj >= 0) ++acnt[find_nz(ri, cj) + 1];
        }
      }
    for (int z = 0; z < nnz; ++z) acnt[z + 1] += acnt[z];
    for (int i = 0; i < N; ++i) fcnt[i + 1] += fcnt[i];
    std::vector<int> alist(acnt[nnz]), flist(fcnt[N]);
    std::vector<int> afill(acnt.begin(), acnt.end() - 1), ffill(fcnt.begin(), fcnt.end() - 1);
    for (int e = 0; e < T; ++e)
      for (int li = 0; li < 12; ++li) {
        const int ri = rows[(size_t)e * 12 + li];
        if (ri < 0) continue;
        flist[ffill[ri]++] = e * 12 + li;
        for (int lj = 0; lj < 12; ++lj) {
          const int cj = rows[(size_t)e * 12 + lj];
          if (cj >= 0) alist[afill[find_nz(ri, cj)]++] = e * 144 + li * 12 + lj;
        }
      }
    f->rows.upload(rows.data(), rows.size());
    f->rp.upload(rp.data(), rp.size());
    f->col.upload(col.data(), col.size());
    f->aptr.upload(acnt.data(), acnt.size());
    f->alist.upload(alist.data(), alist.size());
    f->nzrow.upload(nzrow.data(), nzrow.size());
    f->fptr.upload(fcnt.data(), fcnt.size());
    f->flist.upload(flist.data(), flist.size());
    f->dpos.upload(dpos.data(), dpos.size());
    NL_CUDA(cudaMalloc(&f->isdiag, nnz));
    NL_CUDA(cudaMemcpy(f->isdiag, isd.data(), nnz, cudaMemcpyHostToDevice));
    f->Dm_inv.alloc((size_t)T * 9);
    NL_CUDA(cudaMemcpy(f->Dm_inv.p, d->Dm_inv, (size_t)T * 9 * 8, cudaMemcpyHostToDevice));
    f->vol.alloc(T);
    NL_CUDA(cudaMemcpy(f->vol.p, d->vol, (size_t)T * 8, cudaMemcpyHostToDevice));
    f->mass.alloc(N);
    NL_CUDA(cudaMemcpy(f->mass.p, d->mass, (size_t)N * 8, cudaMemcpyHostToDevice));
    for (DBuf* bf : {&f->u, &f->v, &f->x, &f->up, &f->fext, &f->b, &f->dinv, &f->fint, &f->cg_x, &f->cg_r, &f->cg_z,
                     &f->cg_p, &f->cg_Ap})
      bf->alloc(N);
    f->cg_Ap.alloc((size_t)2 * N);  // Ap | second direction buffer
    f->fe.alloc((size_t)T * 12);
    f->Ke.alloc((size_t)T * 144);
    f->epart.alloc((T + 7) / 8);
    f->Kv.alloc(nnz);
    f->Hv.alloc(nnz);
    f->gpart.alloc((N + 255) / 256);
    f->relres.alloc(1);
    f->iters.alloc(1);
    // cooperative PCG grid: one block per SM (co-residency required by grid.sync)
    int sms = 0, occ = 0;
    NL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    NL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fs_pcg, PCG_NTH, 0));
    if (occ < 1) throw Error(NLROM_ERR_CUDA, "k_fs_pcg cannot be resident");
    // one 1024-thread block per SM (tools/bench_fullspace.py: 37..296 blocks all within 10%)
    f->pcg_blocks = std::max(1, std::min(sms, (N + 31) / 32));
    f->cg_part.alloc((size_t)f->pcg_blocks * 4);
    NL_CUDA(cudaDeviceSynchronize());
    *out = f;
    return NLROM_OK;
  } catch (const Error& e) {
    const int code = e.code;
    nlrom_fs_destroy(f);
    return code;
  }
}

// elements at up -> fe, Ke (if want_K), energy (host sum of the block partials, fixed order)
static double fs_elements(nlrom_fs* f, bool want_K) {
  const int nbk = (f->T + 7) / 8;
  FsElemArgs a{f->rows.p, f->Dm_inv.p, f->vol.p, f->up.p, f->T, f->mu, f->lam, f->fe.p, want_K ? f->Ke.p : nullptr,
               f->epart.p};
  k_fs_elements<<<nbk, 256, 0, f->st>>>(a);
  NL_CHECK_LAUNCH();
  f->hpart.resize(nbk);
  NL_CUDA(cudaMemcpyAsync(f->hpart.data(), f->epart.p, nbk * 8, cudaMemcpyDeviceToHost, f->st));
  NL_CUDA(cudaStreamSynchronize(f->st));
  double s = 0.0;
  for (double v : f->hpart) s += v;
  return s;
}

extern "C" int nlrom_fs_energy_force(nlrom_fs* f, const double* u, double* energy, double* f_int) {
  FS_TRY(f)
  NL_CUDA(cudaMemcpyAsync(f->up.p, u, (size_t)f->N * 8, cudaMemcpyHostToDevice, f->st));
  const double en = fs_elements(f, false);
  if (energy) *energy = en;
  if (f_int) {
    // residual kernel with x = v = f_ext = 0, mass terms vanish: fint = gathered element forces
    NL_CUDA(cudaMemsetAsync(f->x.p, 0, (size_t)f->N * 8, f->st));
    NL_CUDA(cudaMemsetAsync(f->Hv.p, 0, (size_t)f->nnz * 8, f->st));
    k_fs_residual<<<(f->N + 255) / 256, 256, 0, f->st>>>(f->fptr.p, f->flist.p, f->fe.p, f->rp.p, f->col.p, f->Kv.p,
                                                         f->Hv.p, f->dpos.p, f->mass.p, f->x.p, f->x.p, f->x.p, 1.0,
                                                         0.0, 0.0, f->N, f->b.p, f->dinv.p, f->fint.p, f->gpart.p);
    NL_CHECK_LAUNCH();
    NL_CUDA(cudaMemcpyAsync(f_int, f->fint.p, (size_t)f->N * 8, cudaMemcpyDeviceToHost, f->st));
    NL_CUDA(cudaStreamSynchronize(f->st));
  }
  FS_END(f)
}

extern "C" int nlrom_fs_step(nlrom_fs* f, const double* u, const double* v, const double* f_ext,
                             const nlrom_fs_cfg* cfg, double* u_out, double* v_out, nlrom_fs_info* info) {
  FS_TRY(f)
  if (!cfg || !(cfg->dt > 0)) throw Error(NLROM_ERR_ARG, "dt must be > 0 (SPEC.md:346)");
  const int N = f->N;
  const double dt = cfg->dt;
  NL_CUDA(cudaMemcpyAsync(f->u.p, u, (size_t)N * 8, cudaMemcpyHostToDevice, f->st));
  NL_CUDA(cudaMemcpyAsync(f->v.p, v, (size_t)N * 8, cudaMemcpyHostToDevice, f->st));
  NL_CUDA(cudaMemcpyAsync(f->fext.p, f_ext, (size_t)N * 8, cudaMemcpyHostToDevice, f->st));
  NL_CUDA(cudaMemcpyAsync(f->x.p, f->v.p, (size_t)N * 8, cudaMemcpyDeviceToDevice, f->st));  // v' = v initially
  double fn = 0.0;
  for (int i = 0; i < N; ++i) fn += f_ext[i] * f_ext[i];
  const double tol = cfg->newton_tol * std::max(1.0, std::sqrt(fn));
  const int g1 = std::min(2048, (N + 255) / 256);
  const int nres = (N + 255) / 256;
  std::vector<double> gp(nres);
  int it = 0, cg_total = 0;
  double gnorm = 0.0, energy = 0.0;
  for (;;) {
    k_fs_axpy<<<g1, 256, 0, f->st>>>(f->up.p, f->u.p, f->x.p, dt, N);  // u' = u + dt v'
    NL_CHECK_LAUNCH();
    energy = fs_elements(f, true);
    k_fs_assemble<<<std::min(4096, (f->nnz + 255) / 256), 256, 0, f->st>>>(
        f->aptr.p, f->alist.p, f->nzrow.p, f->isdiag, f->Ke.p, f->mass.p, f->beta * dt + dt * dt, 1.0 + f->alpha * dt,
        f->nnz, f->Kv.p, f->Hv.p);
    NL_CHECK_LAUNCH();
    k_fs_residual<<<nres, 256, 0, f->st>>>(f->fptr.p, f->flist.p, f->fe.p, f->rp.p, f->col.p, f->Kv.p, f->Hv.p,
                                          f->dpos.p, f->mass.p, f->x.p, f->v.p, f->fext.p, dt, f->alpha, f->beta, N,
                                          f->b.p, f->dinv.p, f->fint.p, f->gpart.p);
    NL_CHECK_LAUNCH();
    NL_CUDA(cudaMemcpyAsync(gp.data(), f->gpart.p, nres * 8, cudaMemcpyDeviceToHost, f->st));
    NL_CUDA(cudaStreamSynchronize(f->st));
    double g2 = 0.0;
    for (double x : gp) g2 += x;
    gnorm = std::sqrt(g2);
    if (!std::isfinite(gnorm)) throw Error(NLROM_ERR_NONFINITE, "non-finite full-space residual");
    if (gnorm <= tol) break;
    if (it >= cfg->max_iters) {
      char buf[160];
      snprintf(buf, sizeof buf, "full-space Newton did not converge in %d iterations; last residual norm %.3e",
               cfg->max_iters, gnorm);
      throw Error(NLROM_ERR_NEWTON, buf);
    }
    PcgArgs pa{f->rp.p, f->col.p, f->Hv.p, f->dinv.p, f->b.p, f->cg_x.p, f->cg_r.p, f->cg_z.p, f->cg_p.p,
               f->cg_Ap.p, f->cg_part.p, N, cfg->cg_tol, cfg->cg_max_iters, f->iters.p, f->relres.p};
    void* kargs[] = {&pa};
    NL_CUDA(cudaLaunchCooperativeKernel((const void*)k_fs_pcg, dim3(f->pcg_blocks), dim3(PCG_NTH), kargs, 0, f->st));
    int cit = 0;
    NL_CUDA(cudaMemcpyAsync(&cit, f->iters.p, 4, cudaMemcpyDeviceToHost, f->st));
    k_fs_axpy<<<g1, 256, 0, f->st>>>(f->x.p, f->x.p, f->cg_x.p, 1.0, N);  // v' += dv
    NL_CHECK_LAUNCH();
    NL_CUDA(cudaStreamSynchronize(f->st));
    cg_total += cit;
    ++it;
  }
  NL_CUDA(cudaMemcpyAsync(u_out, f->up.p, (size_t)N * 8, cudaMemcpyDeviceToHost, f->st));
  NL_CUDA(cudaMemcpyAsync(v_out, f->x.p, (size_t)N * 8, cudaMemcpyDeviceToHost, f->st));
  NL_CUDA(cudaStreamSynchronize(f->st));
  if (info) {
    info->iters = it;
    info->cg_iters = cg_total;
    info->res_norm = gnorm;
    info->energy = energy;
  }
  FS_END(f)
}
