/* Nearest-neighbour upscale of 28x28 binary digit images to an h x w canvas,
 * emitted as a sorted CSR row per image.  Pure index bookkeeping for the
 * synthetic input generator (sdnngen.ms_inputs); no arithmetic of the method.
 * ys[y] / xs[x] map a target row / column to its source row / column; both are
 * non-decreasing, so emitting target rows in order gives sorted CSR rows. */
#include <stdint.h>

static int64_t row_cols(const uint8_t *srow, int32_t w, const int32_t *xs, int32_t *cols) {
    int64_t c = 0;
    for (int32_t x = 0; x < w; ++x)
        if (srow[xs[x]]) cols[c++] = x;
    return c;
}

/* pass 1: nnz per image (cols: scratch of w int32) */
void ms_count(int64_t B, const uint8_t *img, int32_t h, int32_t w,
              const int32_t *ys, const int32_t *xs, int64_t *nnz_per_img, int32_t *cols) {
    for (int64_t b = 0; b < B; ++b) {
        const uint8_t *im = img + b * 784;
        int64_t c = 0, cur = 0;
        int32_t prev = -1;
        for (int32_t y = 0; y < h; ++y) {
            if (ys[y] != prev) { prev = ys[y]; cur = row_cols(im + prev * 28, w, xs, cols); }
            c += cur;
        }
        nnz_per_img[b] = c;
    }
}

/* pass 2: column indices; rowptr[b] is the absolute write offset of image b in idx */
void ms_fill(int64_t B, const uint8_t *img, int32_t h, int32_t w,
             const int32_t *ys, const int32_t *xs, const int64_t *rowptr, int32_t *idx,
             int32_t *cols) {
    for (int64_t b = 0; b < B; ++b) {
        const uint8_t *im = img + b * 784;
        int32_t *out = idx + rowptr[b];
        int64_t cur = 0;
        int32_t prev = -1;
        for (int32_t y = 0; y < h; ++y) {
            if (ys[y] != prev) { prev = ys[y]; cur = row_cols(im + prev * 28, w, xs, cols); }
            int32_t base = y * w;
            for (int64_t i = 0; i < cur; ++i) *out++ = base + cols[i];
        }
    }
}

/* RadiX-Net butterfly lists: out[c*32 + v] = outer[(inner[c] & ~(31<<p)) | (v<<p)].
 * With outer = pi_l, inner = pi_{l+1}^-1 this is the source list of output c
 * (ELLCOL); with outer = pi_{l+1}, inner = pi_l^-1 the output list of input c
 * (CSR row c).  Index bookkeeping only. */
void rn_lists(int64_t n, int32_t p, const int64_t *outer, const int64_t *inner, int32_t *out) {
    const int64_t mask = ~((int64_t)31 << p);
    for (int64_t c = 0; c < n; ++c) {
        const int64_t base = inner[c] & mask;
        int32_t *o = out + c * 32;
        for (int64_t v = 0; v < 32; ++v) o[v] = (int32_t)outer[base | (v << p)];
    }
}
