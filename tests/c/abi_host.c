/* The C ABI from plain C99 (what a cgo / JNI / FFI binding would compile
 * against): include the header, call the host-only entry points (no GPU
 * needed), check the reference's values and error behaviour. */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "fgb200.h"

static int fails = 0;
#define CHECK(c) do { if (!(c)) { fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++fails; } } while (0)

int main(void) {
    CHECK(fgb_version() >= 10000);
    /* pad_radius: FIR ceil(r*sigma) (min 1), IIR ceil(5 sigma)+2, box 0 (gaussian.py:198-212) */
    fgb_smoother fir = {FGB_SMOOTH_FIR, 0, 3.0}, iir = {FGB_SMOOTH_IIR, 0, 0.0}, box = {FGB_SMOOTH_BOX, 2, 0.0};
    CHECK(fgb_pad_radius(&fir, 4.0) == 12);
    CHECK(fgb_pad_radius(&iir, 4.0) == 22);
    CHECK(fgb_pad_radius(&box, 4.0) == 0);
    /* make_coeffs KAT, sigma = 4: B = sum(a) */
    double c[4];
    CHECK(fgb_iir_coeffs(4.0, c) == FGB_OK);
    CHECK(fabs(c[0] - 0.03780278999660075) < 1e-15 && fabs(c[1] + 2.1629127524845253) < 1e-14);
    CHECK(fabs(c[0] - (1.0 + c[1] + c[2] + c[3])) < 1e-14);
    /* sigma < 0.5 with the IIR is a ValueError in the reference (message mentions ExactFIR) */
    CHECK(fgb_iir_coeffs(0.3, c) == FGB_EINVAL);
    CHECK(strstr(fgb_last_error(), "ExactFIR") != NULL);
    /* sampled_gaussian: 2h+1 taps, unit sum, symmetric */
    double w[64];
    int32_t half = 0;
    CHECK(fgb_sampled_gaussian(2.0, 3.0, w, 64, &half) == FGB_OK);
    CHECK(half == 6);
    double s = 0.0;
    for (int i = 0; i <= 2 * half; ++i) s += w[i];
    CHECK(fabs(s - 1.0) < 1e-15 && w[0] == w[2 * half]);
    CHECK(fgb_sampled_gaussian(2.0, 3.0, w, 4, &half) == FGB_EINVAL);
    /* descriptor validation runs before any device work */
    double om = 1.0, sg = 2.0;
    fgb_bank_desc d;
    memset(&d, 0, sizeof d);
    d.img.height = 0; d.img.width = 8; d.img.pitch = 8; d.img.batch = 1; d.img.dtype = FGB_F32;
    d.n_freq = 1; d.orientations = 4; d.omegas = &om; d.sigmas = &sg; d.smoother = fir; d.reuse = 1;
    CHECK(fgb_bank(&d, NULL, NULL, NULL) == FGB_EINVAL);  /* image dimensions must be at least 1x1 */
    CHECK(strlen(fgb_last_error()) > 0);
    d.img.height = 8;
    CHECK(fgb_bank_entries(&d) == 4);
    sg = -1.0;
    CHECK(fgb_bank(&d, NULL, NULL, NULL) == FGB_EINVAL);  /* sigma must be positive */
    if (fails == 0) printf("abi_host ok\n");
    return fails != 0;
}
