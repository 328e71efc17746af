/* A plain-C consumer of the C ABI (include/pulse_cuda.h): the binding surface a
 * cgo / JNI / N-API host would use.  Builds a two-tensor checkpoint pair, then
 * pulse_encode -> pulse_write_patch_bytes -> pulse_read_patch_bytes ->
 * pulse_decode (hash verified) and checks the result bit for bit; then checks
 * that a truncated patch is rejected with the reference's TruncationError.
 *
 *   gcc -std=c11 -O2 -I include examples/c_abi_roundtrip.c \
 *       -L paper_2602_03839_b200 -lpulse_cuda -Wl,-rpath,$PWD/paper_2602_03839_b200
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pulse_cuda.h"

#define CHECK(call)                                                                       \
    do {                                                                                  \
        pulse_status st_ = (call);                                                        \
        if (st_ != PULSE_OK) {                                                            \
            fprintf(stderr, "%s failed: %d %s\n", #call, (int)st_, pulse_last_error());   \
            return 1;                                                                     \
        }                                                                                 \
    } while (0)

int main(void) {
    enum { R = 300, C = 40, V = 777 };
    static uint16_t a_prev[R * C], a_curr[R * C], b_prev[V], b_curr[V], a_out[R * C], b_out[V];
    uint32_t x = 12345u;
    for (int i = 0; i < R * C; ++i) {
        x = x * 1664525u + 1013904223u;
        a_prev[i] = (uint16_t)(x >> 16);
        a_curr[i] = (x & 31u) == 0 ? (uint16_t)(a_prev[i] ^ 1u) : a_prev[i];
    }
    for (int i = 0; i < V; ++i) {
        x = x * 1664525u + 1013904223u;
        b_prev[i] = (uint16_t)(x >> 16);
        b_curr[i] = (i % 7 == 3) ? (uint16_t)(b_prev[i] + 1u) : b_prev[i];
    }
    int64_t sa[2] = {R, C}, sb[1] = {V};
    pulse_tensor prev_t[2] = {{"layer.a", sa, 2, a_prev, R * C}, {"layer.b", sb, 1, b_prev, V}};
    pulse_tensor curr_t[2] = {{"layer.a", sa, 2, a_curr, R * C}, {"layer.b", sb, 1, b_curr, V}};
    pulse_checkpoint prev = {7, prev_t, 2}, curr = {8, curr_t, 2};

    for (uint32_t repr = PULSE_COO_DOWNSCALED; repr <= PULSE_FLAT_INT32; ++repr) {
        pulse_patch* patch = NULL;
        CHECK(pulse_encode(&curr, &prev, repr, PULSE_ZSTD1, &patch));
        pulse_bytes* wire = NULL;
        CHECK(pulse_write_patch_bytes(patch, &wire));
        pulse_patch* back = NULL;
        CHECK(pulse_read_patch_bytes(pulse_bytes_data(wire), pulse_bytes_size(wire), &back));
        uint16_t* outs[2] = {a_out, b_out};
        uint64_t step = 0;
        CHECK(pulse_decode(&prev, back, 1, outs, &step));
        if (step != 8 || memcmp(a_out, a_curr, sizeof a_out) || memcmp(b_out, b_curr, sizeof b_out)) {
            fprintf(stderr, "repr %u: decoded checkpoint differs\n", repr);
            return 1;
        }
        pulse_patch* bad = NULL;
        const pulse_status st = pulse_read_patch_bytes(pulse_bytes_data(wire), pulse_bytes_size(wire) - 5, &bad);
        if (st == PULSE_OK) {
            fprintf(stderr, "repr %u: truncated patch accepted\n", repr);
            return 1;
        }
        printf("repr %u: %llu-byte patch, round trip exact, truncated patch -> status %d (%s)\n", repr,
               (unsigned long long)pulse_bytes_size(wire), (int)st, pulse_last_error());
        pulse_patch_free(back);
        pulse_bytes_free(wire);
        pulse_patch_free(patch);
    }
    printf("C ABI round trip OK (%s)\n", pulse_version());
    return 0;
}
