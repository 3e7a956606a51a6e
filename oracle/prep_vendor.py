"""Prepare the nlohmann/json header the reference build needs (TEST INFRASTRUCTURE).

The reference (`/root/reference/proj`) vendors nlohmann/json but does not ship
it (`proj/.gitignore:2`, `proj/README.md:13-14`).  The only copy in this image
is cudnn_frontend's v3.11.3, which carries a local patch that prints integer
arrays on one line.  The reference's goldens were produced by stock nlohmann
`dump(2)`, so we restore the stock branch.

Output goes to oracle/_ref/vendor/json.hpp only (git-ignored).
"""
import os
import sys

SRC = ("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/"
       "cudnn_frontend/thirdparty/nlohmann/json.hpp")


def main(out_dir):
    os.makedirs(out_dir, exist_ok=True)
    s = open(SRC).read()
    patched = ("if (pretty_print && (elementType != value_t::number_integer) &&\n"
               "                    (elementType != value_t::number_unsigned))")
    if patched in s:
        s = s.replace(patched, "if (pretty_print)")
        s = s.replace("auto elementType = val.m_data.m_value.array->begin()->type();",
                      "[[maybe_unused]] auto elementType = "
                      "val.m_data.m_value.array->begin()->type();")
    with open(os.path.join(out_dir, "json.hpp"), "w") as f:
        f.write(s)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "oracle/_ref/vendor")
