// Shim TU (test infrastructure, not product): compiles the UNMODIFIED reference
// source /root/reference/proj/core/src/wire.cpp. The reference's `namespace rewind`
// collides with glibc's `void rewind(FILE*)` (stdio.h), so the standard library
// is included first under its real name and the namespace is renamed for the
// reference TU only. See SURVEY.md §8(c).
#include <bits/stdc++.h>
#define rewind rewind_ref
#include "/root/reference/proj/core/src/wire.cpp"
