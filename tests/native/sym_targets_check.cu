// Host-side check (tests/test_sym_layout_host.py): the constant-period sym_targets_g used by the
// PSF epilogue equals the generic sym_targets of the symmetric tile layout for every block.
#include "dwc_internal.cuh"
#include <cstdio>
using namespace dwc;
int main() {
    long bad = 0, n = 0;
    for (int g : {1, 2, 4})
        for (int T = 1; T <= 120; T++)
            for (int a = 0; a < T; a++)
                for (int b = 0; b < T; b++) {
                    int t0[3], t1[3];
                    const int n0 = sym_targets(T, g, a, b, t0), n1 = sym_targets_g(T, g, a, b, t1);
                    n++;
                    if (n0 != n1) { bad++; continue; }
                    for (int u = 0; u < n0; u++) bad += t0[u] != t1[u];
                }
    printf("checked %ld, mismatches %ld\n", n, bad);
    return bad != 0;
}
