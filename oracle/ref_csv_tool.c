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
int ref_checkpoint_roundtrip(const char*, const char*);
int ref_output_dir_name(int, int, int, double, int, int, char*, int);
int ref_write_densities(const int64_t*, const uint64_t*, int, int, const char*, int);

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
    if (!strcmp(argv[1], "roundtrip") && argc == 4) return ref_checkpoint_roundtrip(argv[2], argv[3]);
    if (!strcmp(argv[1], "dirname") && argc == 8) {
        char buf[256];
        int rc = ref_output_dir_name(atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), strtod(argv[5], 0), atoi(argv[6]),
                                     atoi(argv[7]), buf, 256);
        puts(buf);
        return rc;
    }
    if (!strcmp(argv[1], "densities") && argc >= 6) { /* densities <path> <append> <S> mcs c0..cS ... */
        int append = atoi(argv[3]), S = atoi(argv[4]);
        int n = (argc - 5) / (S + 2);
        int64_t* st = malloc(sizeof(int64_t) * (n + 1));
        uint64_t* c = malloc(sizeof(uint64_t) * (n + 1) * (S + 1));
        for (int i = 0; i < n; ++i) {
            st[i] = strtoll(argv[5 + i * (S + 2)], 0, 10);
            for (int v = 0; v <= S; ++v) c[i * (S + 1) + v] = strtoull(argv[6 + i * (S + 2) + v], 0, 10);
        }
        return ref_write_densities(st, c, n, S, argv[2], append);
    }
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
