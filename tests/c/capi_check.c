/* Plain-C consumer of include/soaforge_b200.h: proves the header is valid C
 * and the library links and behaves like the reference ABI on the host-side
 * entries (test_capi.cpp semantics).  Prints "capi ok" on success. */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "soaforge_b200.h"

#define CHECK(c)                                                     \
    do {                                                             \
        if (!(c)) {                                                  \
            printf("FAIL %s:%d %s (%s)\n", __FILE__, __LINE__, #c,  \
                   sf_last_error());                                 \
            return 1;                                                \
        }                                                            \
    } while (0)

int main(void) {
    int s = 0, e = 0, m = 0;
    double q = 0;
    uint64_t bits = 0;
    int fields = 0;
    const char* text = NULL;
    sf_schema* h = NULL;
    sf_schema* again = NULL;
    sf_config* cfg = NULL;
    sf_view* v = NULL;

    CHECK(sf_version() && strlen(sf_version()) > 0);
    CHECK(sf_layout_for(32, &s, &e, &m) == SF_OK && s == 1 && e == 8 && m == 23);
    CHECK(sf_layout_for(6, &s, &e, &m) == SF_INVALID_ARG && strlen(sf_last_error()) > 0);
    CHECK(sf_layout_for(16, NULL, &e, &m) == SF_INVALID_ARG);
    CHECK(sf_quantize(3.14159265358979312, 17, &q) == SF_OK && q == 3.140625);
    CHECK(sf_quantize(1.0, 99, &q) == SF_INVALID_ARG);

    CHECK(sf_schema_parse("schema s { field a : f64 x3; field b : f32 @truncate(20); }", &h) == SF_OK);
    CHECK(sf_schema_record_bits(h, &bits) == SF_OK && bits == 192 + 20);
    CHECK(sf_schema_field_count(h, &fields) == SF_OK && fields == 2);
    CHECK(sf_schema_print(h, &text) == SF_OK);
    CHECK(sf_schema_parse(text, &again) == SF_OK);
    CHECK(sf_schema_record_bits(again, &bits) == SF_OK && bits == 212);
    sf_schema_destroy(again);
    again = NULL;
    CHECK(sf_schema_parse("schema { oops", &again) == SF_PARSE_ERROR && again == NULL);

    CHECK(sf_b200_view_create(h, NULL, SF_LAYOUT_SOA, SF_PREC_NATIVE, "", 100, &v) == SF_OK);
    CHECK(sf_b200_view_bytes(v, &bits) == SF_OK && bits == 100 * (3 * 64 + 32) / 8);
    sf_b200_view_destroy(v);
    sf_schema_destroy(h);

    CHECK(sf_config_create(&cfg) == SF_OK);
    CHECK(sf_config_set_int(cfg, "particles", 128) == SF_OK);
    CHECK(sf_config_set_int(cfg, "particles", -1) == SF_INVALID_ARG);
    CHECK(sf_config_set_string(cfg, "variants", "cpu-baseline,dev-soa") == SF_OK);
    CHECK(sf_config_set_string(cfg, "writeback", "sometimes") == SF_INVALID_ARG);
    CHECK(sf_config_set_double(cfg, "bandwidth", 0.0) == SF_INVALID_ARG);
    sf_config_destroy(cfg);
    printf("capi ok\n");
    return 0;
}
