#!/bin/bash
# Mutation check for the oracle pins: each call applies one plausible slip to
# oracle/oracle.c in a scratch copy and reports how many oracle pins fail.
# Usage: tests/oracle_mutations.sh   (runs the list at the bottom; ~30 s)
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WORK=$(mktemp -d); cd "$WORK"
mut() {
# apply a sed mutation to oracle.c, rebuild into a temp copy of the repo, run the oracle pins
name=$1; shift
rm -rf repo && mkdir repo && cp -r "$ROOT"/oracle "$ROOT"/synth "$ROOT"/tests repo/
rm -f repo/oracle/liboracle.so
sed -i "$@" repo/oracle/oracle.c
if cmp -s repo/oracle/oracle.c "$ROOT"/oracle/oracle.c; then echo "$name: MUTATION DID NOT APPLY"; exit; fi
cd repo && res=$(python -m pytest tests/test_oracle.py -q -m "not gpu" -p no:cacheprovider 2>&1 | tail -1)
echo "$name: $res"
cd "$WORK"
}
mut old_L_in_apply 's/double l = (\*Lij + /double Lo = *Lij; double l = (*Lij + /; s/\*Vj = c \* (\*Vj) - s \* l;/*Vj = c * (*Vj) - s * Lo;/'
mut drop_sigma_apply 's/double l = (\*Lij + (double)sigma \* s \* (\*Vj)) \/ c;/double l = (*Lij + s * (*Vj)) \/ c;/'
mut drop_sigma_compute 's/double x = d \* d + (double)sigma \* (Vi \* Vi);/double x = d * d + (Vi * Vi);/'
mut s_over_w 's/\*s = Vi \/ d;/*s = Vi \/ w;/'
mut c_inverted 's/\*c = w \/ d;/*c = d \/ w;/'
mut printed_order_A 's/        for (int64_t j = 0; j < i; ++j)$/        for (int64_t j = 0; j < 0; ++j)/'
mut e_loop_wrong_index 's/gcmo_apply(cs_c\[j \* k + e\], cs_s\[j \* k + e\]/gcmo_apply(cs_c[j * k + 0], cs_s[j * k + 0]/'
mut transposed_L 's/#define LIJ(i, j) L\[(size_t)(i) + (size_t)(j) \* (size_t)ldl\]/#define LIJ(i, j) L[(size_t)(j) + (size_t)(i) * (size_t)ldl]/'
mut fail_nonstrict 's/int bad = !(x > 0.0);/int bad = !(x >= 0.0);/'
rm -rf "$WORK"
