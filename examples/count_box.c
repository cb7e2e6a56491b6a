/*
 * count_box.c -- the whole-box counting functions from C through the library's
 * own communicator (include/eis.h, "the whole box"): one process per GPU.
 *
 *   RANK, WORLD_SIZE, LOCAL_RANK   as torchrun / mpirun set them (default 0, 1, 0)
 *   EIS_ID_FILE                    path through which rank 0 hands the NCCL id to
 *                                  the other ranks (default /tmp/eis_comm_id)
 *   argv: lo x_1 ... x_n           counts over lo < d <= x_i
 *
 * Prints one JSON line per rank: {"rank":r,"world":G,"lo":lo,"x":[...],"D":[...],"E":[...]}.
 * pi_D(x), pi_E(x) are PAPER.md l.105-108's counting functions (lo = 0).
 *
 * Build: gcc -O2 -I include examples/count_box.c -L paper_2507_06579_b200 -leis \
 *            -Wl,-rpath,$PWD/paper_2507_06579_b200 -o count_box
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "eis.h"

static int env_int(const char *k, int dflt) {
    const char *v = getenv(k);
    return v && *v ? atoi(v) : dflt;
}

static int die(const char *what, int rc) {
    fprintf(stderr, "%s failed (%d): %s\n", what, rc, eis_last_error());
    return 1;
}

int main(int argc, char **argv) {
    if (argc < 3) {
        fprintf(stderr, "usage: %s lo x_1 [x_2 ...]\n", argv[0]);
        return 2;
    }
    const int rank = env_int("RANK", 0), world = env_int("WORLD_SIZE", 1);
    const int local = env_int("LOCAL_RANK", 0);
    const char *idf = getenv("EIS_ID_FILE") ? getenv("EIS_ID_FILE") : "/tmp/eis_comm_id";
    const uint64_t lo = strtoull(argv[1], NULL, 10);
    const size_t n = (size_t)(argc - 2);
    uint64_t *x = malloc(n * sizeof *x), *cD = malloc(n * sizeof *cD), *cE = malloc(n * sizeof *cE);
    for (size_t i = 0; i < n; i++) x[i] = strtoull(argv[2 + i], NULL, 10);

    int rc = eis_init(local);
    if (rc) return die("eis_init", rc);
    unsigned char id[EIS_COMM_ID_BYTES];
    if (rank == 0) {                                   /* publish the id atomically */
        if ((rc = eis_comm_unique_id(id))) return die("eis_comm_unique_id", rc);
        char tmp[4096];
        snprintf(tmp, sizeof tmp, "%s.tmp", idf);
        FILE *f = fopen(tmp, "wb");
        if (!f || fwrite(id, 1, sizeof id, f) != sizeof id || fclose(f) || rename(tmp, idf)) {
            perror("id file");
            return 1;
        }
    } else {                                           /* wait for it */
        FILE *f = NULL;
        for (int t = 0; t < 600 && !(f = fopen(idf, "rb")); t++) usleep(100000);
        if (!f || fread(id, 1, sizeof id, f) != sizeof id) {
            fprintf(stderr, "no NCCL id in %s\n", idf);
            return 1;
        }
        fclose(f);
    }
    if ((rc = eis_comm_init(id, world, rank))) return die("eis_comm_init", rc);
    if ((rc = eis_count_window_comm(lo, x, n, cD, cE))) return die("eis_count_window_comm", rc);
    printf("{\"rank\":%d,\"world\":%d,\"lo\":%llu,\"x\":[", rank, world, (unsigned long long)lo);
    for (size_t i = 0; i < n; i++) printf("%s%llu", i ? "," : "", (unsigned long long)x[i]);
    printf("],\"D\":[");
    for (size_t i = 0; i < n; i++) printf("%s%llu", i ? "," : "", (unsigned long long)cD[i]);
    printf("],\"E\":[");
    for (size_t i = 0; i < n; i++) printf("%s%llu", i ? "," : "", (unsigned long long)cE[i]);
    printf("]}\n");
    eis_comm_finalize();
    eis_finalize();
    free(x);
    free(cD);
    free(cE);
    return 0;
}
