/* Exhaustive pin of the oracle's hand-written fp32 -> fp16 RNE conversion
 * against the compiler's IEEE binary16 conversion (_Float16, round to
 * nearest even) over all 2^32 fp32 bit patterns.  NaNs are compared by
 * class (both NaN, same sign).  Test helper only; links liboracle.so. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

uint16_t orc_f32_to_f16(float x);
float orc_f16_to_f32(uint16_t h);

int main(void)
{
    uint64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+:bad)
    for (int64_t i = 0; i <= 0xffffffffll; ++i) {
        uint32_t u = (uint32_t)i;
        float x; memcpy(&x, &u, 4);
        uint16_t mine = orc_f32_to_f16(x);
        _Float16 ref = (_Float16)x;
        uint16_t rb; memcpy(&rb, &ref, 2);
        int mine_nan = (mine & 0x7c00) == 0x7c00 && (mine & 0x3ff);
        int ref_nan = (rb & 0x7c00) == 0x7c00 && (rb & 0x3ff);
        int ok = (mine_nan || ref_nan) ? (mine_nan && ref_nan && ((mine ^ rb) & 0x8000) == 0)
                                       : mine == rb;
        if (!ok) {
            if (bad < 10) printf("MISMATCH x=0x%08x mine=0x%04x ref=0x%04x\n", u, mine, rb);
            bad++;
        }
    }
    /* fp16 -> fp32 widening: all 2^16 patterns against the compiler. */
    for (uint32_t h = 0; h < 65536; ++h) {
        uint16_t hb = (uint16_t)h;
        _Float16 hv; memcpy(&hv, &hb, 2);
        float ref = (float)hv, mine = orc_f16_to_f32(hb);
        uint32_t a, b; memcpy(&a, &ref, 4); memcpy(&b, &mine, 4);
        int nan = ref != ref;
        int ok = nan ? (mine != mine && ((a ^ b) & 0x80000000u) == 0) : a == b;
        if (!ok && bad++ < 20)
            printf("WIDEN MISMATCH h=0x%04x mine=0x%08x ref=0x%08x\n", h, b, a);
    }
    printf("mismatches=%llu\n", (unsigned long long)bad);
    return bad != 0;
}
