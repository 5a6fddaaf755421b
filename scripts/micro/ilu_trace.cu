// Trace of the level-scheduled sync-free sweep on a 27-point nx^3 grid:
// per row, globaltimer at grab / dependencies ready / done.
#include <cuda/atomic>
#include <algorithm>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int ld_relaxed(int *p) {
    cuda::atomic_ref<int, cuda::thread_scope_device> a(*p);
    return a.load(cuda::memory_order_relaxed);
}
constexpr int kFS = 32;

template <int WAIT>
__global__ void k_sweep(int n, const int *order, const int *ptr, const int *col, const int *dpos,
                        const double *lu, double *y, int *flags, int *counter,
                        unsigned long long *tr) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n) return;
        const unsigned long long t0 = gtime();
        const int i = order[t];
        const int b = ptr[i], e = dpos[i];
        if (WAIT == 0) {  // lane 0 sequential
            if (lane == 0) {
                for (int j = e - 1; j >= b; --j) {
                    int *f = flags + (long long)col[j] * kFS;
                    while (ld_relaxed(f) == 0) {}
                }
                cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
            }
            __syncwarp();
        } else {  // parallel test, lane 0 spins on one pending
            for (;;) {
                int pend = -1;
                for (int j = b + lane; j < e; j += 32) {
                    const int k = col[j];
                    if (ld_relaxed(flags + (long long)k * kFS) == 0) { pend = k; break; }
                }
                const unsigned m = __ballot_sync(0xffffffffu, pend >= 0);
                if (!m) break;
                const int k = __shfl_sync(0xffffffffu, pend, __ffs(m) - 1);
                if (lane == 0) while (ld_relaxed(flags + (long long)k * kFS) == 0) {}
                __syncwarp();
            }
            cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
            __syncwarp();
        }
        const unsigned long long t1 = gtime();
        double acc = 0.0;
        if (lane < 3) acc = y[3LL * i + lane];
        for (int c = b; c < e; c += 32) {
            const int j = c + lane;
            double x0 = 0, x1 = 0, x2 = 0;
            if (j < e) { const double *g = y + 3LL * col[j]; x0 = __ldcg(g); x1 = __ldcg(g + 1); x2 = __ldcg(g + 2); }
            const int m = min(32, e - c);
            for (int d = 0; d < m; ++d) {
                const double v0 = __shfl_sync(0xffffffffu, x0, d), v1 = __shfl_sync(0xffffffffu, x1, d),
                             v2 = __shfl_sync(0xffffffffu, x2, d);
                if (lane < 3) {
                    const double *bl = lu + 9LL * (c + d) + 3 * lane;
                    acc = __dsub_rn(acc, __dmul_rn(bl[0], v0));
                    acc = __dsub_rn(acc, __dmul_rn(bl[1], v1));
                    acc = __dsub_rn(acc, __dmul_rn(bl[2], v2));
                }
            }
        }
        if (lane < 3) y[3LL * i + lane] = acc;
        __syncwarp();
        if (lane == 0) {
            cuda::atomic_ref<int, cuda::thread_scope_device> a(flags[(long long)i * kFS]);
            a.store(1, cuda::memory_order_release);
            const unsigned long long t2 = gtime();
            tr[3LL * i] = t0; tr[3LL * i + 1] = t1; tr[3LL * i + 2] = t2;
        }
    }
}

int main(int argc, char **argv) {
    const int nx = argc > 1 ? atoi(argv[1]) : 40;
    const int n = nx * nx * nx;
    std::vector<int> ptr(n + 1, 0), col, dpos(n);
    for (int z = 0; z < nx; ++z) for (int yy = 0; yy < nx; ++yy) for (int x = 0; x < nx; ++x) {
        const int i = (z * nx + yy) * nx + x;
        for (int dz = -1; dz <= 1; ++dz) for (int dy = -1; dy <= 1; ++dy) for (int dx = -1; dx <= 1; ++dx) {
            const int X = x + dx, Y = yy + dy, Z = z + dz;
            if (X < 0 || Y < 0 || Z < 0 || X >= nx || Y >= nx || Z >= nx) continue;
            const int k = (Z * nx + Y) * nx + X;
            if (k == i) dpos[i] = (int)col.size();
            col.push_back(k);
        }
        ptr[i + 1] = (int)col.size();
    }
    std::vector<int> lev(n), ord(n);
    int maxl = 0;
    for (int i = 0; i < n; ++i) { int l = 0; for (int j = ptr[i]; j < dpos[i]; ++j) l = std::max(l, lev[col[j]] + 1); lev[i] = l; maxl = std::max(maxl, l); }
    std::vector<int> cnt(maxl + 2, 0);
    for (int i = 0; i < n; ++i) ++cnt[lev[i] + 1];
    for (int l = 0; l <= maxl; ++l) cnt[l + 1] += cnt[l];
    for (int i = 0; i < n; ++i) ord[cnt[lev[i]]++] = i;
    const long long nnz = col.size();
    int *dptr, *dcol, *ddpos, *dord, *flags, *counter; double *lu, *y; unsigned long long *tr;
    cudaMalloc(&dptr, 4 * (n + 1)); cudaMalloc(&dcol, 4 * nnz); cudaMalloc(&ddpos, 4 * n); cudaMalloc(&dord, 4 * n);
    cudaMalloc(&flags, 4LL * n * kFS + 4); cudaMalloc(&counter, 4); cudaMalloc(&lu, 72 * nnz); cudaMalloc(&y, 24LL * n);
    cudaMalloc(&tr, 24LL * n);
    cudaMemcpy(dptr, ptr.data(), 4 * (n + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(dcol, col.data(), 4 * nnz, cudaMemcpyHostToDevice);
    cudaMemcpy(ddpos, dpos.data(), 4 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dord, ord.data(), 4 * n, cudaMemcpyHostToDevice);
    cudaMemset(lu, 0, 72 * nnz); cudaMemset(y, 0, 24LL * n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("nx %d n %d levels %d\n", nx, n, maxl + 1);
    for (int wait = 0; wait < 2; ++wait)
        for (int per : {1, 2, 4}) {
            cudaMemset(flags, 0, 4LL * n * kFS + 4); cudaMemset(counter, 0, 4);
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            if (wait == 0) k_sweep<0><<<sms * per, 256>>>(n, dord, dptr, dcol, ddpos, lu, y, flags, counter, tr);
            else k_sweep<1><<<sms * per, 256>>>(n, dord, dptr, dcol, ddpos, lu, y, flags, counter, tr);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            std::vector<unsigned long long> h(3LL * n);
            cudaMemcpy(h.data(), tr, 24LL * n, cudaMemcpyDeviceToHost);
            double wait_s = 0, work_s = 0;
            for (int i = 0; i < n; ++i) { wait_s += h[3 * i + 1] - h[3 * i]; work_s += h[3 * i + 2] - h[3 * i + 1]; }
            printf("wait-mode %d ctas/sm %d: %.3f ms = %.2f us/level; per row: wait %.2f us, work %.2f us (%s)\n",
                   wait, per, ms, 1e3 * ms / (maxl + 1), wait_s / n / 1e3, work_s / n / 1e3,
                   cudaGetErrorString(cudaGetLastError()));
        }
}
