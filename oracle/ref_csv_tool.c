/* ref_csv_tool — runs the reference's CSV writers (experiments.cpp:242-285) out of process.
 *   *** TEST INFRASTRUCTURE ONLY ***   (oracle/_ref/ref_csv_tool, linked against libescg_ref.so)
 *   ref_csv_tool extinction <path> <t0> <c0> <t1> <c1> ...
 *   ref_csv_tool coexistence <path> <trials> <coexisting> <probability> <mobility> <length> <mcs>
 *   ref_csv_tool format <double>...                                         (format_double) */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

int ref_write_extinction_csv(const int64_t*, const int*, int, const char*);
int ref_write_coexistence_csv(int, int, double, double, int, int64_t, const char*);
int ref_format_double(double, char*, int);

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    if (!strcmp(argv[1], "extinction")) {
        int n = (argc - 3) / 2;
        int64_t* t = malloc(sizeof(int64_t) * (n + 1));
        int* c = malloc(sizeof(int) * (n + 1));
        for (int i = 0; i < n; ++i) {
            t[i] = strtoll(argv[3 + 2 * i], 0, 10);
            c[i] = atoi(argv[4 + 2 * i]);
        }
        return ref_write_extinction_csv(t, c, n, argv[2]);
    }
    if (!strcmp(argv[1], "coexistence") && argc == 9)
        return ref_write_coexistence_csv(atoi(argv[3]), atoi(argv[4]), strtod(argv[5], 0), strtod(argv[6], 0),
                                         atoi(argv[7]), strtoll(argv[8], 0, 10), argv[2]);
    if (!strcmp(argv[1], "format")) {
        char buf[64];
        for (int i = 2; i < argc; ++i) {
            ref_format_double(strtod(argv[i], 0), buf, 64);
            puts(buf);
        }
        return 0;
    }
    return 2;
}
