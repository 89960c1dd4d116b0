# SASS of one kernel from a built object: tools/sass_of.sh <object> <mangled-name-substring>
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : /{p = index($0, pat) > 0} p'
